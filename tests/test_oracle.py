"""CPU: the oracle pinned against the golden fixtures and the SPEC.md
known-answer examples; the three restatements agree with each other."""
import os

import numpy as np
import pytest

from oracle import seq, taskbench_np as tnp, tokens as T
from paper_2508_16522_b200.flat import IntervalCSR, transpose
from paper_2508_16522_b200.taskbench import generate_graph

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
from golden.make_golden import CASES  # noqa: E402


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracles_match_golden(case):
    name, pat, W, Tn, kind, arg, seed, P = case
    g = generate_graph(pat, W, Tn, n_workers=P, mapping="round_robin", kind=kind, arg=arg)
    want = GOLD[name]
    np.testing.assert_array_equal(seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=seed), want)
    np.testing.assert_array_equal(tnp.run(pat, W, Tn, seed=seed, kind=kind, arg=arg), want)
    st = GOLD[name + "__stats"]
    assert st[0] == g.cross_worker_edges()


def test_python_oracle_matches_golden():
    g = generate_graph("stencil_1d", 8, 100)
    got = seq.run_py(g.n, [g.pred.row(v) for v in range(g.n)], seed=0)
    np.testing.assert_array_equal(np.array(got, dtype=np.uint64), GOLD["stencil_8x100_s0"])


def test_affine_map_equals_literal_loop():
    rng = np.random.default_rng(0)
    for n in [0, 1, 2, 3, 7, 64, 100, 1000, 4097]:
        x = int(rng.integers(0, 2**63))
        a, c = T.affine_pow(n)
        assert (a * x + c) & T.M64 == T.lcg_iter_int(x, n)
    for n in [0, 1, 5, 33]:
        h = int(rng.integers(0, 2**63))
        assert T.compute_body_int(h, n) == seq.compute_loop(h, n)
        assert int(T.compute_body(np.array([h], np.uint64), n)[0]) == T.compute_body_int(h, n)


def test_mix64_vector_equals_scalar():
    xs = np.array([0, 1, 2**63, 2**64 - 1, 0x9E3779B97F4A7C15], dtype=np.uint64)
    assert [int(v) for v in T.mix64(xs)] == [T.mix64_int(int(x)) for x in xs]


@pytest.mark.parametrize("pat,W,Tn,nodes,edges", [
    ("stencil", 8, 2, 16, 22),
    ("independent", 4, 3, 12, 0),
    ("stencil", 1, 5, 5, 4),
    ("stencil", 8, 100, 800, 2178),       # BASELINE configs[0]
    ("no_comm", 1024, 1000, 1024000, 1022976),
    ("stencil_1d", 1024, 1000, 1024000, 3066930),
    ("tree", 4096, 1000, 4050943, 4050942),
    ("nearest", 8192, 100, 819200, 4054446),
    ("all_to_all", 8192, 10, 81920, 603979776),
])
def test_generate_graph_counts(pat, W, Tn, nodes, edges):
    g = generate_graph(pat, W, Tn)
    assert (g.n, g.n_edges()) == (nodes, edges)
    assert g.succ.n_edges() == edges


@pytest.mark.slow
def test_fft_counts():
    g = generate_graph("fft", 4096, 1000)
    assert (g.n, g.n_edges()) == (4096000, 11595928)


@pytest.mark.parametrize("pat", ["stencil_1d", "stencil_1d_periodic", "fft", "tree", "nearest", "no_comm",
                                 "spread", "all_to_all", "trivial"])
def test_successors_are_transpose(pat):
    for W, Tn in [(1, 3), (2, 4), (13, 9), (64, 7), (16, 1), (1, 1)]:   # (T = 1: no edges at all)
        g = generate_graph(pat, W, Tn)
        s = transpose(g.pred)
        assert np.array_equal(s.ptr, g.succ.ptr) and np.array_equal(s.iv, g.succ.iv)


@pytest.mark.parametrize("pat", ["stencil_1d", "fft", "tree", "nearest", "no_comm", "spread", "all_to_all"])
def test_single_step_graphs(pat):
    """T = 1: every task is a source (an early version failed to pack the empty rows)."""
    g = generate_graph(pat, 16, 1, n_workers=4)
    assert g.n_edges() == 0 and g.succ.n_edges() == 0
    np.testing.assert_array_equal(seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=3),
                                  tnp.run(pat, 16, 1, seed=3))


def test_interval_csr_roundtrip():
    rows = [[], [0], [0, 1, 2], [5, 7, 8, 9]]
    c = IntervalCSR.from_lists(10, rows + [[]] * 6)
    assert [c.row(v) for v in range(4)] == [[], [0], [0, 1, 2], [5, 7, 8, 9]]
    assert c.iv.tolist() == [[0, 0], [0, 2], [5, 5], [7, 9]]


def test_column_checksums():
    tok = GOLD["stencil_8x100_s0"]
    cs = tnp.column_checksums("stencil_1d", 8, 100, tok)
    assert np.array_equal(cs, T.column_checksums(tok, 8))


def test_oracle_affine_map_matches_literal_loop():
    """The oracle's affine shortcut equals the literal loop (the pin for the
    long-body GPU checks in test_gpu_parity.py)."""
    g = generate_graph("no_comm", 4, 2, kind=2, arg=1000)
    a = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=3)
    b = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=3, literal_loop=True)
    np.testing.assert_array_equal(a, b)


def test_memory_bound_body_three_restatements():
    """MEMORY(n) (memory_bound): C, numpy and pure-Python oracles agree."""
    g = generate_graph("stencil_1d", 6, 4, kind=T.BODY_MEMORY, arg=192)
    c = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=5)
    p = np.array(seq.run_py(g.n, [g.pred.row(v) for v in range(g.n)], g.kind, g.arg, seed=5), dtype=np.uint64)
    np.testing.assert_array_equal(c, p)
    h = np.array([1, 2, 3], dtype=np.uint64)
    r = T.memory_body(h, np.array([64, 128, 0]))
    assert int(r[0]) == T.memory_body_int(1, 64) and int(r[1]) == T.memory_body_int(2, 128) and int(r[2]) == 0
