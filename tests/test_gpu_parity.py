"""GPU parity: the persistent executor vs the sequential oracles, bit-exact,
through the C ABI (include/tdexec.h)."""
import numpy as np
import pytest

from paper_2508_16522_b200 import _native as N
from paper_2508_16522_b200.executor import DeviceGraph, device_info
from paper_2508_16522_b200.flat import FlatGraph, IntervalCSR, transpose
from paper_2508_16522_b200.taskbench import generate_graph
from oracle import seq, taskbench_np as tnp

pytestmark = pytest.mark.gpu


def _oracle(g, seed):
    return seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=seed, order=None if g.order is None else np.argsort(g.order))


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_stencil_8x100(seed):
    g = generate_graph("stencil_1d", 8, 100, n_workers=8)
    with DeviceGraph(g) as dg:
        dg.run(seed=seed, flags=N.TD_F_CHECKSUM | N.TD_F_TALLY | N.TD_F_STATS)
        got = dg.tokens()
        np.testing.assert_array_equal(got, _oracle(g, seed))
        np.testing.assert_array_equal(got, tnp.run("stencil_1d", 8, 100, seed=seed))
        np.testing.assert_array_equal(dg.checksums(), tnp.column_checksums("stencil_1d", 8, 100, got))
        assert (dg.tally() == 1).all()
        st = dg.stats()
        assert st["executed"] == 800
        assert st["cross_worker_edges"] == g.cross_worker_edges()


@pytest.mark.parametrize("pattern,W,T,kind,arg", [
    ("no_comm", 64, 50, 0, 0), ("stencil_1d", 100, 30, 2, 5), ("fft", 64, 30, 0, 0),
    ("tree", 64, 20, 2, 3), ("nearest", 50, 20, 0, 0), ("all_to_all", 40, 6, 0, 0),
    ("spread", 32, 10, 0, 0), ("stencil_1d_periodic", 16, 10, 0, 0), ("trivial", 10, 3, 0, 0),
    ("all_to_all", 300, 3, 2, 2),
])
@pytest.mark.parametrize("mapping,workers", [("block", None), ("round_robin", 7), ("block", 3)])
def test_patterns(pattern, W, T, kind, arg, mapping, workers):
    g = generate_graph(pattern, W, T, n_workers=workers, mapping=mapping, kind=kind, arg=arg)
    with DeviceGraph(g) as dg:
        dg.run(seed=11)
        np.testing.assert_array_equal(dg.tokens(), _oracle(g, 11))


def test_replay_idempotent_epochs():
    # many replays on one uploaded graph (epoch-scaled counters, no reset)
    g = generate_graph("stencil_1d", 32, 20, n_workers=32)
    want = {s: _oracle(g, s) for s in (0, 5)}
    with DeviceGraph(g) as dg:
        for i in range(50):
            s = 0 if i % 2 == 0 else 5
            dg.run(seed=s, flags=N.TD_F_TALLY)
            np.testing.assert_array_equal(dg.tokens(), want[s])
            assert (dg.tally() == 1).all()


def test_queued_launches_back_to_back():
    g = generate_graph("fft", 128, 40)
    with DeviceGraph(g) as dg:
        for _ in range(20):
            dg.launch(seed=3, flags=N.TD_F_QUEUE)
        dg.wait()
        np.testing.assert_array_equal(dg.tokens(), _oracle(g, 3))


@pytest.mark.parametrize("pattern,W,T,workers", [("stencil_1d", 64, 30, 64), ("fft", 4096, 12, 4096), ("tree", 256, 20, 64)])
def test_checksum_banks(pattern, W, T, workers):
    """Column checksums alternate between two device banks by checksum-launch
    parity (no memset before the kernel): every launch's checksums equal the
    oracle's, a launch without TD_F_CHECKSUM leaves the last checksums
    readable, and queued checksum launches each fold into their own bank."""
    g = generate_graph(pattern, W, T, n_workers=workers)
    want = {s: tnp.column_checksums(pattern, W, T, _oracle(g, s)) for s in (1, 2, 3)}
    with DeviceGraph(g) as dg:
        for i in range(7):
            s = 1 + i % 3
            dg.run(seed=s, flags=N.TD_F_CHECKSUM)
            np.testing.assert_array_equal(dg.checksums(), want[s])
        dg.run(seed=1, flags=0)                      # no checksum: bank of seed 1 (i = 6) still current
        np.testing.assert_array_equal(dg.checksums(), want[1])
        dg.run(seed=2, flags=N.TD_F_CHECKSUM | N.TD_F_STATS)   # the diagnostics kernel zeroes banks too
        np.testing.assert_array_equal(dg.checksums(), want[2])
        for s in (3, 1, 2, 3):
            dg.launch(seed=s, flags=N.TD_F_QUEUE | N.TD_F_CHECKSUM)
        dg.wait()
        np.testing.assert_array_equal(dg.checksums(), want[3])
        dg.run(seed=1, flags=N.TD_F_CHECKSUM)
        np.testing.assert_array_equal(dg.checksums(), want[1])


def test_random_dags():
    rng = np.random.default_rng(0)
    for trial in range(100):
        n = int(rng.integers(1, 65))
        preds = []
        for v in range(n):
            k = int(rng.integers(0, min(v, 6) + 1)) if v else 0
            preds.append(sorted(rng.choice(v, size=k, replace=False).tolist()) if k else [])
        # random permutation of ids so id order is NOT topological
        perm = rng.permutation(n)
        pr = [[int(perm[u]) for u in preds[v]] for v in range(n)]
        rows = [None] * n
        for v in range(n):
            rows[perm[v]] = pr[v]
        pred = IntervalCSR.from_lists(n, rows)
        succ = transpose(pred)
        P = int(rng.integers(1, 5))
        kind = rng.choice([0, 2], size=n).astype(np.uint8)
        arg = rng.integers(0, 4, size=n).astype(np.uint32)
        g = FlatGraph(n=n, pred=pred, succ=succ, kind=kind, arg=arg,
                      worker=rng.integers(0, P, size=n).astype(np.int32), n_workers=P)
        with DeviceGraph(g) as dg:
            dg.run(seed=trial, flags=N.TD_F_TALLY)
            want = np.array(seq.run_py(n, [pred.row(v) for v in range(n)], kind, arg, seed=trial), dtype=np.uint64)
            np.testing.assert_array_equal(dg.tokens(), want)
            assert (dg.tally() == 1).all()


def test_device_info():
    info = device_info(0)
    assert info["sm_count"] >= 100
    assert info["max_workers"] >= 1024


@pytest.mark.parametrize("pattern,W,T,kind,arg", [
    ("stencil_1d", 1024, 1000, 2, 1),     # BASELINE configs[1] (full size)
    ("no_comm", 1024, 1000, 2, 1),
    ("fft", 4096, 1000, 0, 0),            # configs[2]
    ("tree", 4096, 1000, 0, 0),
    ("nearest", 8192, 100, 0, 0),         # configs[3] (single-GPU form)
    ("all_to_all", 8192, 10, 0, 0),
])
def test_full_size_configs(pattern, W, T, kind, arg):
    info = device_info(0)
    g = generate_graph(pattern, W, T, n_workers=min(W, info["max_workers"]), kind=kind, arg=arg)
    with DeviceGraph(g) as dg:
        dg.run(seed=1, flags=N.TD_F_TALLY | N.TD_F_CHECKSUM)
        dg.run(seed=2, flags=N.TD_F_TALLY | N.TD_F_CHECKSUM)   # second epoch on the same upload
        got = dg.tokens()
        want = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=2)
        np.testing.assert_array_equal(got, want)
        assert (dg.tally() == 1).all()
        np.testing.assert_array_equal(dg.checksums(), tnp.column_checksums(pattern, W, T, got))


def test_golden_fixtures_on_gpu():
    import os
    from golden.make_golden import CASES
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    for name, pat, W, T, kind, arg, seed, P in CASES:
        g = generate_graph(pat, W, T, n_workers=P, mapping="round_robin", kind=kind, arg=arg)
        with DeviceGraph(g) as dg:
            dg.run(seed=seed, flags=N.TD_F_STATS)
            np.testing.assert_array_equal(dg.tokens(), gold[name])
            st = dg.stats()
            assert st["cross_worker_edges"] == gold[name + "__stats"][0]
            assert st["local_decrements"] == gold[name + "__stats"][1]


def test_set_body_arg_reparameterises_in_place():
    g = generate_graph("stencil_1d", 64, 30, kind=2, arg=1)
    with DeviceGraph(g) as dg:
        for it in (1, 7, 0, 33):
            dg.set_body_arg(it)
            dg.run(seed=2)
            g.arg[:] = it
            np.testing.assert_array_equal(dg.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=2))


@pytest.mark.parametrize("pattern,W,T,mapping,workers", [
    ("stencil_1d", 256, 20, "block", None), ("fft", 128, 16, "round_robin", 40), ("nearest", 96, 12, "block", 24),
    ("no_comm", 64, 30, "block", 16)])
def test_plain_and_general_kernels_agree(pattern, W, T, mapping, workers, monkeypatch):
    """Graphs that qualify for the PLAIN one-GPU kernel give the same tokens on
    it and on the general kernel (TD_NO_PLAIN, read at upload)."""
    g = generate_graph(pattern, W, T, n_workers=workers, mapping=mapping, kind=2, arg=3)
    want = _oracle(g, 5)
    for no_plain in (False, True):
        if no_plain:
            monkeypatch.setenv("TD_NO_PLAIN", "1")
        else:
            monkeypatch.delenv("TD_NO_PLAIN", raising=False)
        with DeviceGraph(g) as dg:
            for flags in (0, N.TD_F_CHECKSUM, N.TD_F_STATS):
                dg.run(seed=5, flags=flags)
                np.testing.assert_array_equal(dg.tokens(), want)


@pytest.mark.parametrize("pattern,W,T,workers,kind,arg", [
    ("stencil_1d", 64, 20, 16, 2, 3), ("stencil_1d", 1024, 50, 128, 2, 1), ("no_comm", 64, 30, 32, 2, 2),
    ("nearest", 96, 12, 24, 0, 0), ("fft", 128, 16, 32, 2, 1), ("stencil_1d", 40, 10, 20, 0, 0),
    ("nearest", 8192, 10, 2048, 0, 0), ("fft", 4096, 12, 2048, 2, 1)])
def test_group_mode(pattern, W, T, workers, kind, arg, monkeypatch):
    """Multi-column workers (block mapping) run in GROUP mode -- K = 4 nodes
    per warp pass when every list splits into equal-level 4-groups, else K = 2
    (PAIR) -- and give the oracle's tokens, with and without checksums.  The
    mode actually selected is asserted (td_graph_info_get); TD_GROUP=2 caps K
    at 2 and TD_NO_PAIR (read at upload) forces the one-node loop, which must
    agree."""
    g = generate_graph(pattern, W, T, n_workers=workers, mapping="block", kind=kind, arg=arg)
    cols = W // workers
    for mode, env in ((4 if cols % 4 == 0 else 2, {}), (2, {"TD_GROUP": "2"}), (0, {"TD_NO_PAIR": "1"})):
        for k in ("TD_GROUP", "TD_NO_PAIR"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with DeviceGraph(g) as dg:
            assert dg.info()["group"] == mode, (mode, env)
            for seed, flags in ((5, 0), (6, N.TD_F_CHECKSUM)):
                dg.run(seed=seed, flags=flags)
                got = dg.tokens()
                np.testing.assert_array_equal(got, _oracle(g, seed))
                if flags:
                    np.testing.assert_array_equal(dg.checksums(), tnp.column_checksums(pattern, W, T, got))


@pytest.mark.parametrize("env", [{}, {"TD_GROUP": "2"}, {"TD_NO_PAIR": "1"}])
def test_group_ring_slot_wrap(env, monkeypatch):
    """Ring aliasing inside one warp pass: on a single worker whose list is
    4 chains x 17 levels (positions 4l + c), the node at position 1 also feeds
    position 64 -- ring delta 63, so its add lands in ring slot 0, the slot of
    position 0 of the SAME group.  That slot must be consumed before the add
    (tdexec.cu execute_group / execute_node); tokens are checked on the GROUP-4,
    PAIR and one-node loops."""
    for k in ("TD_GROUP", "TD_NO_PAIR"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    L, C = 17, 4
    n = L * C
    rows = [[] if p < C else [p - C] for p in range(n)]
    rows[64] = sorted([1, 60])
    pred = IntervalCSR.from_lists(n, rows)
    g = FlatGraph(n=n, pred=pred, succ=transpose(pred), kind=np.full(n, 2, np.uint8),
                  arg=np.full(n, 3, np.uint32), worker=np.zeros(n, np.int32), n_workers=1)
    g.order = np.arange(n, dtype=np.int64)
    want = np.array(seq.run_py(n, [pred.row(v) for v in range(n)], g.kind, g.arg, seed=4), dtype=np.uint64)
    with DeviceGraph(g) as dg:
        assert dg.info()["group"] == (0 if "TD_NO_PAIR" in env else int(env.get("TD_GROUP", 4)))
        for _ in range(3):
            dg.run(seed=4)
            np.testing.assert_array_equal(dg.tokens(), want)


@pytest.mark.parametrize("iters", [1 << 6, 1 << 10, 1 << 14, 1 << 20, (1 << 20) + 5])
@pytest.mark.parametrize("pattern,W,T,workers", [("stencil_1d", 64, 6, 64), ("no_comm", 64, 4, 32)])
def test_compute_bound_long_bodies(iters, pattern, W, T, workers):
    """compute_bound at the long end of the METG sweep (2^6 .. 2^20 iterations,
    SPEC.md:527-535): the real LCG loop on the GPU against the oracle's O(1)
    affine map, on the one-node and the PAIR loops."""
    g = generate_graph(pattern, W, T, n_workers=workers, mapping="block", kind=2, arg=1)
    with DeviceGraph(g) as dg:
        dg.set_body_arg(iters)
        dg.run(seed=9, flags=N.TD_F_CHECKSUM)
        g.arg[:] = iters
        got = dg.tokens()
        np.testing.assert_array_equal(got, _oracle(g, 9))
        np.testing.assert_array_equal(dg.checksums(), tnp.column_checksums(pattern, W, T, got))



@pytest.mark.parametrize("pattern,W,T,words,workers", [
    ("stencil_1d", 64, 10, 64, 64), ("no_comm", 128, 6, 4096, 32), ("fft", 64, 8, 65536, 64),
    ("tree", 64, 8, 1024, 16)])
def test_memory_bound_body(pattern, W, T, words, workers):
    """memory_bound (TD_BODY_MEMORY, SPEC.md:161-164 / Task Bench): each task
    streams `words` u64 through its worker's scratch and folds them back;
    tokens bit-exact against the C oracle, on one- and multi-column workers."""
    from paper_2508_16522_b200.errors import CompileError, ContractViolation
    g = generate_graph(pattern, W, T, n_workers=workers, mapping="block", kind=6, arg=words)
    with DeviceGraph(g) as dg:
        with pytest.raises(ContractViolation):
            dg.run(seed=1)                       # no scratch attached
        dg.attach_scratch(words)
        for seed in (1, 2):
            dg.run(seed=seed, flags=N.TD_F_CHECKSUM)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, seed))
    g.arg[:] = 100                               # not a multiple of 64
    with pytest.raises(CompileError):
        DeviceGraph(g)


@pytest.mark.parametrize("pattern,W,T,workers,want_group", [
    ("tree", 4096, 30, 2048, 2), ("tree", 4096, 30, 1024, 4), ("tree", 256, 20, 64, 4)])
def test_padded_group_layout(pattern, W, T, workers, want_group, monkeypatch):
    """Worker lists whose equal-level runs are ragged (tree: the first levels
    are narrower than the worker count) are padded with empty slots to whole
    GROUP groups; the padded layout gives the oracle's tokens on the GROUP
    kernel, on the diagnostics kernel (exactly-once tally, executed == n), and
    TD_NO_PAD restores the one-node loop."""
    monkeypatch.delenv("TD_GROUP", raising=False)
    monkeypatch.delenv("TD_NO_PAIR", raising=False)
    g = generate_graph(pattern, W, T, n_workers=workers, mapping="block", kind=2, arg=2)
    for nopad in (False, True):
        if nopad:
            monkeypatch.setenv("TD_NO_PAD", "1")
        with DeviceGraph(g) as dg:
            info = dg.info()
            if not nopad:
                assert info["group"] == want_group and info["n_positions"] > g.n
            else:
                assert info["n_positions"] == g.n
            dg.run(seed=3, flags=N.TD_F_CHECKSUM)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, 3))
            dg.run(seed=4, flags=N.TD_F_TALLY | N.TD_F_STATS)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, 4))
            assert (dg.tally() == 1).all()
            assert dg.stats()["executed"] == g.n
    monkeypatch.delenv("TD_NO_PAD", raising=False)


@pytest.mark.parametrize("W,T,workers,kind,arg,env", [
    (4096, 4, 4096, 0, 0, {}),                                        # default policy: 8 replicas, 1 producer per worker
    (2048, 4, 1024, 0, 0, {"TD_COMBINE": "1"}),                       # 4 replicas, 2 producers per worker, forced
    (1100, 5, 1100, 2, 3, {"TD_COMBINE": "1"}),                       # 3 replicas, forced
    (600, 3, 300, 1, 200, {"TD_COMBINE": "1", "TD_SHARE_FANOUT": "64"}),  # 10 replicas, busy_wait bodies
    (8192, 3, 4096, 0, 0, {"TD_SHARE_FANOUT": "1024"}),
])
def test_bundled_combiners(W, T, workers, kind, arg, env, monkeypatch):
    """Bundled groups with combiner words (tdexec.cu COMB_MIN_REP): producers add
    into a combiner, the completing add forwards (k << 48) + partial sum to every
    replica.  Tokens, exactly-once and re-arming across replays against the oracle
    and against the same graph lowered without combiners."""
    for k in ("TD_COMBINE", "TD_SHARE_FANOUT"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = generate_graph("all_to_all", W, T, n_workers=workers, kind=kind, arg=arg)
    with DeviceGraph(g) as dg:
        assert dg.info()["n_combiners"] > 0
        for seed in (1, 2, 3):
            dg.run(seed=seed, flags=N.TD_F_CHECKSUM | N.TD_F_TALLY | N.TD_F_STATS)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, seed))
            assert (dg.tally() == 1).all()
        dg.run(seed=4, flags=0)
        got = dg.tokens()
    monkeypatch.setenv("TD_COMBINE", "0")
    with DeviceGraph(g) as dg:
        assert dg.info()["n_combiners"] == 0
        dg.run(seed=4, flags=0)
        np.testing.assert_array_equal(dg.tokens(), got)


def test_combiner_policy(monkeypatch):
    """Default policy: no combiners when a worker produces more than two nodes
    of a bundled group (the returning add would serialise its nodes)."""
    for k in ("TD_COMBINE", "TD_SHARE_FANOUT"):
        monkeypatch.delenv(k, raising=False)
    with DeviceGraph(generate_graph("all_to_all", 8192, 2, n_workers=2048)) as dg:
        assert dg.info()["n_combiners"] == 0
    with DeviceGraph(generate_graph("all_to_all", 8192, 2, n_workers=4096)) as dg:
        assert dg.info()["n_combiners"] == 128  # one group (level 1): 8192 producers / 64
    with DeviceGraph(generate_graph("all_to_all", 2048, 2, n_workers=2048)) as dg:
        assert dg.info()["n_combiners"] == 0  # 4 replicas


@pytest.mark.parametrize("pattern,W,T,workers", [("stencil_1d", 1024, 1, 1024), ("no_comm", 8192, 1, 2048),
                                                 ("nearest", 8192, 2, 2048), ("all_to_all", 256, 1, 64),
                                                 ("fft", 64, 1, 16), ("stencil_1d", 8, 2, 8)])
def test_one_and_two_step_graphs(pattern, W, T, workers):
    """Graphs of one or two levels (sources only / one edge layer), every kernel variant they lower to."""
    g = generate_graph(pattern, W, T, n_workers=workers, kind=2, arg=3)
    with DeviceGraph(g) as dg:
        for seed, fl in ((1, 0), (2, N.TD_F_CHECKSUM), (3, N.TD_F_TALLY | N.TD_F_STATS)):
            dg.run(seed=seed, flags=fl)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, seed))


@pytest.mark.parametrize("fanin", [2, 3, 4])
def test_group_ring_rounds(fanin, monkeypatch):
    """GROUP passes whose nodes feed the same ring slots (tdexec.cu: upload-coloured
    rounds of plain shared-memory adds, DF_RING_ROUND_SHIFT).  Worker 0 holds 4
    columns per level; node (l, c) takes its inputs from `fanin` nodes of level
    l - 1 of the SAME worker (all ring-fed), so up to 4 nodes of a pass add into
    one slot and the pass needs up to 4 rounds.  In the second graph worker 1
    holds 4 chains and feeds column 0 of worker 0 at every level: worker 0's
    passes then wait on L2 anyway, and their ring-fed nodes are demoted to
    mailboxes (TD_MIXED_RING=1 keeps them)."""
    for k in ("TD_GROUP", "TD_NO_PAIR", "TD_MIXED_RING"):
        monkeypatch.delenv(k, raising=False)
    L, C = 20, 4
    for mixed in (False, True):
        n0 = L * C
        n = n0 * (2 if mixed else 1)
        rows = []
        for p in range(n0):
            lvl, c = divmod(p, C)
            rows.append([] if lvl == 0 else sorted({(lvl - 1) * C + (c + j) % C for j in range(fanin)}))
        worker = np.zeros(n, np.int32)
        if mixed:  # worker 1: 4 chains; its column 0 of level l also feeds (l + 1, 0) of worker 0
            for p in range(n0):
                lvl, c = divmod(p, C)
                rows.append([] if lvl == 0 else [n0 + (lvl - 1) * C + c])
                worker[n0 + p] = 1
            for lvl in range(1, L):
                rows[lvl * C] = sorted(rows[lvl * C] + [n0 + (lvl - 1) * C])
        pred = IntervalCSR.from_lists(n, rows)
        g = FlatGraph(n=n, pred=pred, succ=transpose(pred), kind=np.full(n, 2, np.uint8),
                      arg=np.full(n, 3, np.uint32), worker=worker, n_workers=2 if mixed else 1)
        key = np.array([((v % n0) // C) * 2 + (v >= n0) for v in range(n)])
        g.order = np.argsort(np.argsort(key, kind="stable"), kind="stable").astype(np.int64)  # rank of each node
        want = np.array(seq.run_py(n, [pred.row(v) for v in range(n)], g.kind, g.arg, seed=5), dtype=np.uint64)
        for keep in ("0", "1"):
            monkeypatch.setenv("TD_MIXED_RING", keep)
            with DeviceGraph(g) as dg:
                assert dg.info()["group"] == 4
                for _ in range(3):
                    dg.run(seed=5)
                    np.testing.assert_array_equal(dg.tokens(), want)
