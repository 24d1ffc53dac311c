"""Sharded replay (PAPER §5 lowering) with several shards on ONE
GPU: every shard is its own persistent kernel on its own stream, and the
cross-shard edges are the same peer-memory atomics the multi-GPU path uses
(same-device peer pointers).  Covers the MULTI kernels -- relays for bundled
groups, rank-tagged successors, the start handshake, the sharded tile body --
on a single-GPU box; tests/test_implicit.py and tests/tools/mgpu_check.py run the
same paths across GPUs."""
import numpy as np
import pytest

from paper_2508_16522_b200 import _native as N
from paper_2508_16522_b200.shard import InProcessShards, ShardingPlan, lowering_stats
from paper_2508_16522_b200.taskbench import generate_graph, generate_stencil2d

pytestmark = pytest.mark.gpu


def _oracle(g, seed):
    from oracle import seq
    return seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=seed)


@pytest.mark.parametrize("pattern,W,T,shards", [
    ("stencil_1d", 256, 30, 2), ("nearest", 240, 12, 3), ("fft", 256, 16, 4), ("tree", 128, 10, 2),
    ("all_to_all", 96, 4, 3), ("all_to_all", 600, 4, 2), ("all_to_all", 1100, 3, 4), ("spread", 192, 8, 2),
    # 8 shards: shard 7's targets carry tag 8 in bits 28..31 (the sign bit of the int32 id)
    ("stencil_1d", 256, 20, 8), ("nearest", 320, 10, 8), ("all_to_all", 1024, 3, 8)])
def test_sharded_same_device(pattern, W, T, shards):
    g = generate_graph(pattern, W, T, n_workers=W)
    sh = InProcessShards(g, ShardingPlan.blocks(W, shards), [0] * shards)
    try:
        for seed in (1, 2, 3):
            sh.run(seed, flags=N.TD_F_TALLY | N.TD_F_STATS, spin_limit=1 << 26)
            np.testing.assert_array_equal(sh.tokens(), _oracle(g, seed))
            for r, d in enumerate(sh.shards):
                mine = sh.node_rank == r
                assert (d.tally()[mine] == 1).all()
        executed = sum(d.stats()["executed"] for d in sh.shards)
        assert executed == g.n
        # without diagnostics: the plain (PLAIN where the shard qualifies) kernels
        sh.run(7, flags=0, spin_limit=1 << 26)
        np.testing.assert_array_equal(sh.tokens(), _oracle(g, 7))
    finally:
        sh.close()


def test_relay_aggregates_cross_shard_messages(monkeypatch):
    """all_to_all on 2 shards: with relays each shard sends one add per remote
    replica per step instead of one per (producer, remote replica)."""
    W, T = 1024, 4
    g = generate_graph("all_to_all", W, T, n_workers=W)
    counts = {}
    for relay in ("0", "1"):
        monkeypatch.setenv("TD_RELAY", relay)
        sh = InProcessShards(g, ShardingPlan.blocks(W, 2), [0, 0])
        try:
            sh.run(5, flags=N.TD_F_STATS, spin_limit=1 << 26)
            np.testing.assert_array_equal(sh.tokens(), _oracle(g, 5))
            counts[relay] = sum(d.stats()["cross_rank_edges"] for d in sh.shards)
        finally:
            sh.close()
    ls = lowering_stats(g, np.repeat(np.arange(2), W // 2)[np.arange(g.n) % W])
    assert ls["ext_pairs"] > 0
    # direct: every producer messages the other shard's replica(s); relayed:
    # one message per (step, shard, remote replica)
    assert counts["0"] == (T - 1) * W
    assert counts["1"] == (T - 1) * 2
    assert counts["1"] < counts["0"]


@pytest.mark.parametrize("mapping", ["block", "shard_block", "shard_cyclic"])
def test_sharded_stencil2d_same_device(mapping):
    from oracle import seq
    nx, ny, T, shards = 512, 768, 4, 3
    ntile = (nx // 64) * (ny // 64)
    g = generate_stencil2d(nx, ny, T, n_workers=ntile // 2, mapping=mapping, shards=shards)
    sh = InProcessShards(g, ShardingPlan.blocks(g.n_workers, shards), [0] * shards, stencil2d=(nx, ny))
    try:
        sh.run(9, flags=N.TD_F_TALLY, spin_limit=1 << 26)
        want_tok, want_grid = seq.stencil2d_tokens(g, seed=9)
        np.testing.assert_array_equal(sh.tokens(), want_tok)
        grid = np.zeros_like(want_grid)
        for r, d in enumerate(sh.shards):
            gr = d.stencil2d_grid((T - 1) & 1)
            for tile in np.unique(np.flatnonzero(sh.node_rank == r) % ntile):
                ty, tx = divmod(int(tile), nx // 64)
                grid[ty * 64:(ty + 1) * 64, tx * 64:(tx + 1) * 64] = gr[ty * 64:(ty + 1) * 64, tx * 64:(tx + 1) * 64]
        np.testing.assert_array_equal(grid, want_grid)
    finally:
        sh.close()


@pytest.mark.parametrize("pattern,W,T,shards,k", [
    ("stencil_1d", 256, 41, 2, 4), ("stencil_1d", 192, 30, 3, 3), ("nearest", 240, 20, 2, 4),
    ("nearest", 384, 25, 3, 2), ("stencil_1d", 512, 60, 4, 8), ("stencil_1d", 512, 40, 8, 4)])
def test_halo_replicas_same_device(pattern, W, T, shards, k):
    """halo-replicated sharded replay: real tokens equal the oracle's, every
    replica computes the token of the node it replicates, all exactly once"""
    g = generate_graph(pattern, W, T, n_workers=W, kind=2, arg=2)
    sh = InProcessShards(g, ShardingPlan.blocks(W, shards), [0] * shards, halo=k)
    try:
        assert sh.halo is not None
        n2 = sh.halo.graph.n
        for seed, flags in ((1, N.TD_F_TALLY), (4, N.TD_F_TALLY), (6, 0)):
            sh.run(seed, flags=flags, spin_limit=1 << 26)
            want = _oracle(g, seed)
            np.testing.assert_array_equal(sh.tokens(), want)
            for r, d in enumerate(sh.shards):
                mine = np.flatnonzero(sh.node_rank == r)
                if flags:
                    assert (d.tally()[mine] == 1).all()
                rep = mine[mine >= g.n]
                np.testing.assert_array_equal(d.tokens()[rep], want[sh.halo.ident[rep]])
        assert n2 > g.n
    finally:
        sh.close()


@pytest.mark.parametrize("pattern,W,T,shards,cols,halo", [
    ("nearest", 512, 12, 2, 4, 0), ("stencil_1d", 256, 30, 4, 2, 0), ("fft", 256, 16, 2, 4, 0),
    ("nearest", 512, 40, 2, 4, 8), ("stencil_1d", 512, 40, 2, 4, 16)])
def test_sharded_group_mode(pattern, W, T, shards, cols, halo):
    """Sharded PLAIN graphs with several columns per worker run the MULTI
    GROUP kernel: groups whose nodes are all shard-local take the K-node pass,
    groups touching the shard boundary (or a successor pool row) run node by
    node on the sharded path.  Tokens bit-exact, exactly-once."""
    g = generate_graph(pattern, W, T, n_workers=W // cols, kind=2, arg=2)
    sh = InProcessShards(g, ShardingPlan.blocks(g.n_workers, shards), [0] * shards, halo=halo)
    try:
        if not halo:
            assert all(d.info()["group"] > 0 for d in sh.shards)
        for seed, flags in ((1, 0), (2, N.TD_F_CHECKSUM), (3, N.TD_F_TALLY | N.TD_F_STATS)):
            sh.run(seed, flags=flags, spin_limit=1 << 26)
            np.testing.assert_array_equal(sh.tokens(), _oracle(g, seed))
        gx = sh.halo.graph if sh.halo is not None else g
        assert sum(d.stats()["executed"] for d in sh.shards) == gx.n
    finally:
        sh.close()
