"""Halo replication of a sharded lowering (shard.replicate_halo), checked on
the CPU: the extended graph, evaluated with each replica hashing as the node
it replicates (td_csr.ident), must reproduce the oracle's tokens, and every
edge that crosses shards must leave a node at a level that is a multiple of
k (the NVLink hop is paid once per k levels)."""
import numpy as np
import pytest

from oracle import seq
from oracle import tokens as T
from paper_2508_16522_b200.flat import kahn_levels
from paper_2508_16522_b200.shard import ShardingPlan, node_shards, replicate_halo
from paper_2508_16522_b200.taskbench import generate_graph


def _eval(g, ident, seed):
    """tokens of a graph whose node v computes node ident[v] (Kahn order)"""
    preds = [g.pred.row(v) for v in range(g.n)]
    succs = [[] for _ in range(g.n)]
    indeg = [len(p) for p in preds]
    for v, p in enumerate(preds):
        for u in p:
            succs[u].append(v)
    ready = [v for v in range(g.n) if indeg[v] == 0]
    tok = [None] * g.n
    while ready:
        v = ready.pop()
        tok[v] = T.token_int(seed, int(ident[v]), [(int(ident[u]), tok[u]) for u in preds[v]],
                             int(g.kind[v]), int(g.arg[v]))
        for s in succs[v]:
            indeg[s] -= 1
            if indeg[s] == 0:
                ready.append(s)
    assert all(t is not None for t in tok)
    return np.array(tok, dtype=np.uint64)


@pytest.mark.parametrize("pattern,W,T_,shards,k", [
    ("stencil_1d", 24, 13, 2, 4), ("stencil_1d", 30, 12, 3, 3), ("stencil_1d", 16, 9, 4, 2),
    ("nearest", 30, 10, 3, 4), ("fft", 16, 9, 2, 3), ("tree", 16, 8, 2, 3), ("spread", 24, 7, 2, 2),
    ("no_comm", 16, 6, 2, 4)])
def test_halo_reproduces_tokens(pattern, W, T_, shards, k):
    g = generate_graph(pattern, W, T_, n_workers=W, kind=2, arg=3)
    plan = ShardingPlan.blocks(W, shards)
    hg = replicate_halo(g, plan, k, max_frac=0.9)
    want = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=5)
    if pattern == "no_comm":  # nothing crosses shards: nothing to replicate
        assert hg is None
        return
    assert hg is not None and hg.graph.n > g.n
    g2, ident = hg.graph, hg.ident
    tok = _eval(g2, ident, seed=5)
    np.testing.assert_array_equal(tok[:g.n], want)
    np.testing.assert_array_equal(tok[g.n:], want[ident[g.n:]])
    # in-degrees preserved; every replica owned by (and run on) one shard
    assert (g2.pred.degrees() == g.pred.degrees()[ident]).all()
    assert (node_shards(g2, hg.plan) == hg.node_rank).all()
    # replicas never replicate local nodes
    own = node_shards(g, plan)
    assert (own[ident[g.n:]] != hg.node_rank[g.n:]).all()
    # cross-shard edges only from nodes at levels that are multiples of k
    lev = kahn_levels(g.pred, g.succ)
    dst, src = g2.pred.expand()
    cross = hg.node_rank[src] != hg.node_rank[dst]
    assert (lev[ident[src[cross]]] % k == 0).all()


def test_halo_declines_dense_and_single_shard():
    g = generate_graph("all_to_all", 64, 6, n_workers=64)
    assert replicate_halo(g, ShardingPlan.blocks(64, 2), 4) is None      # would replicate everything
    g = generate_graph("stencil_1d", 16, 6, n_workers=16)
    assert replicate_halo(g, ShardingPlan.blocks(16, 1), 4) is None      # nothing to shard
    assert replicate_halo(g, ShardingPlan.blocks(16, 2), 1) is None      # k < 2 is no halo


def test_halo_stencil_counts():
    """stencil_1d on 2 shards, period k: at a level L of phase q = L mod k > 0
    each shard replicates the other's boundary cone, min(L - q + k, T - 1) - L
    columns wide (k-1, k-2, ..., 1 across a full period)."""
    k = 4
    for T_ in (41, 43, 45):
        g = generate_graph("stencil_1d", 32, T_, n_workers=32)
        hg = replicate_halo(g, ShardingPlan.blocks(32, 2), k, max_frac=0.5)
        want = sum(max(0, min(L - L % k + k, T_ - 1) - L) for L in range(T_) if L % k)
        assert hg.graph.n - g.n == 2 * want
