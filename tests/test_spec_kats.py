"""CPU: SPEC.md known-answer examples and invariants on the CPU reference
executor (Alg. 1 on taskdual.machine), the graph IR, and compute_metg."""
import numpy as np
import pytest

from oracle import alg1_cpu, seq, substrate
from paper_2508_16522_b200.errors import GraphError
from paper_2508_16522_b200.graph import ExtPostcond, ExtPrecond, Task, build, owners
from paper_2508_16522_b200.metg import Sample, compute_metg
from paper_2508_16522_b200.taskbench import generate_graph

needs_ref = pytest.mark.skipif(not substrate.available(), reason="taskdual.machine not installed")

DIAMOND_NODES = [Task(1, 1), Task(2, 2), Task(1, 3), Task(2, 4)]  # f1@P1 f2@P2 f3@P1 f4@P2
DIAMOND_EDGES = [(0, 1), (0, 2), (1, 3), (2, 3)]


def test_build_diamond_valid():
    g = build(DIAMOND_NODES, DIAMOND_EDGES)
    assert g.n == 4 and len(g.edges) == 4


def test_build_cycle_rejected():
    with pytest.raises(GraphError):
        build(DIAMOND_NODES, DIAMOND_EDGES + [(3, 0)])


def test_build_ext_precond_with_incoming_edge_rejected():
    with pytest.raises(GraphError):
        build([Task(0, 1), ExtPrecond(0)], [(0, 1)])


def test_build_ext_postcond_with_outgoing_edge_rejected():
    with pytest.raises(GraphError):
        build([ExtPostcond(0), Task(0, 1)], [(0, 1)])


def test_build_dangling_and_duplicate_rejected():
    with pytest.raises(GraphError):
        build([Task(0, 1)], [(0, 5)])
    with pytest.raises(GraphError):
        build([Task(0, 1), Task(0, 1)], [(0, 1), (0, 1)])


def test_random_dags_validation_soundness():
    """build accepts iff the graph is a DAG vs brute force."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(1, 12))
        m = int(rng.integers(0, 20))
        e = {(int(a), int(b)) for a, b in rng.integers(0, n, size=(m, 2)) if a != b}
        adj = {v: [b for a, b in e if a == v] for v in range(n)}
        state = [0] * n

        def dfs(v):
            state[v] = 1
            for w in adj[v]:
                if state[w] == 1 or (state[w] == 0 and dfs(w)):
                    return True
            state[v] = 2
            return False
        cyclic = any(state[v] == 0 and dfs(v) for v in range(n))
        try:
            build([Task(0, 1)] * n, sorted(e))
            assert not cyclic
        except GraphError:
            assert cyclic


def test_compile_diamond_owners():  # SPEC.md:376 / 586: P1 {f1,f3}, P2 {f2,f4}
    g = build(DIAMOND_NODES, DIAMOND_EDGES)
    own, rs = owners(g)
    assert rs == [("proc", 1), ("proc", 2)]
    assert own.tolist() == [0, 1, 0, 1]
    indeg = g.pred.degrees().tolist()
    assert indeg == [0, 1, 1, 2]


@needs_ref
def test_alg1_diamond_message_stats():
    tok, st, _ = alg1_cpu.run_flat(4, [[], [0], [0], [1, 2]], [0, 1, 0, 1])
    assert st == dict(cross_worker_messages=2, local_decrements=2, init_messages=2)
    want = seq.run_py(4, [[], [0], [0], [1, 2]])
    assert tok.tolist() == want


@needs_ref
def test_alg1_single_node():
    tok, st, _ = alg1_cpu.run_flat(1, [[]], [0])
    assert st["cross_worker_messages"] == 0 and st["init_messages"] == 1


@needs_ref
def test_alg1_stencil_8x16_round_robin_100_replays():
    g = generate_graph("stencil", 8, 16, n_workers=4, mapping="round_robin")
    rows = [g.pred.row(v) for v in range(g.n)]
    m, e, _ = substrate.load()
    with m.create_machine(m.MachineSpec(processor_count=4)) as mach:
        cg = alg1_cpu.compile_flat(mach, g.n, rows, g.worker)
        for _ in range(100):
            cg.execute(3)
            cg.wait(30)
            st = cg.message_stats()
            assert st["cross_worker_messages"] == 210 == g.cross_worker_edges()
            assert st["local_decrements"] == 120
    assert g.n_edges() == 330


@needs_ref
def test_alg1_forced_interleaving_exactly_once():
    m, e, _ = substrate.load()
    rows = [[], [0], [0], [1, 2]]
    with m.create_machine(m.MachineSpec(processor_count=2)) as mach:
        cg = alg1_cpu.compile_flat(mach, 4, rows, [0, 1, 0, 1])
        w = cg.workers[1]
        fired = []
        w.cg.rt.send_message = lambda aid, mid, payload=None: fired.append((aid, mid, payload))
        w.decrement(3)   # f3's arrival first
        assert fired == []
        w.decrement(3)   # then f2's
        assert fired == [(1, alg1_cpu.EXECUTE_OP, 3)]
        assert w.ctr[3] == 2  # re-armed


@needs_ref
def test_alg1_random_dags_equal_sequential_oracle():
    rng = np.random.default_rng(2)
    for trial in range(150):
        n = int(rng.integers(1, 65))
        rows = [sorted(rng.choice(v, size=int(rng.integers(0, min(v, 5) + 1)), replace=False).tolist())
                if v else [] for v in range(n)]
        P = int(rng.integers(1, 5))
        owner = rng.integers(0, P, size=n)
        kind = rng.choice([0, 2], size=n).astype(np.uint8)
        arg = rng.integers(0, 5, size=n).astype(np.uint32)
        tok, st, _ = alg1_cpu.run_flat(n, rows, owner, kind=kind, arg=arg, seed=trial, processors=P)
        assert tok.tolist() == seq.run_py(n, rows, kind, arg, seed=trial)
        cross = sum(1 for v in range(n) for u in rows[v] if owner[u] != owner[v])
        assert st["cross_worker_messages"] == cross


def test_compute_metg_kat():
    r = compute_metg([(1e3, .10), (1e4, .40), (1e5, .80), (1e6, .99)], 0.5)
    assert r.metg_ns == 1e5


def test_compute_metg_none_and_single():
    assert compute_metg([(1e3, .1), (1e4, .2)], 0.5).metg_ns is None
    assert compute_metg([(7.0, .9)], 0.5).metg_ns == 7.0


def test_compute_metg_from_rates_and_monotone():
    s = [Sample(granularity_ns=g, wall_ns=1, rate=r) for g, r in [(1, 1.0), (2, 3.0), (4, 6.0), (8, 8.0)]]
    a = compute_metg(s, 0.7).metg_ns
    b = compute_metg(s, 0.3).metg_ns
    assert a == 4 and b == 2 and a >= b
    assert compute_metg(s, 0.5).peak_rate == 8.0


def test_compute_metg_fixed_peak():
    """With a fixed reference peak (the chip's), efficiency is rate / peak
    for every sample, not rate / the sweep's best."""
    s = [Sample(granularity_ns=g, wall_ns=0, rate=r) for g, r in [(1e3, 1.0), (1e4, 3.0), (1e5, 6.0)]]
    r = compute_metg(s, 0.5, peak=10.0)
    assert r.peak_is_reference and r.peak_rate == 10.0
    assert [round(x.efficiency, 3) for x in r.curve] == [0.1, 0.3, 0.6]
    assert r.metg_ns == 1e5
    assert compute_metg(s, 0.5).metg_ns == 1e4          # SPEC.md:552 (best measured) for comparison
    assert compute_metg(s, 0.5, peak=20.0).metg_ns is None


def test_cpu_reference_metg_sweep_small():
    """The CPU reference's METG sweep (Alg. 1 on taskdual.machine, C bodies),
    every point checked against the oracle."""
    from oracle import alg1_cpu, seq
    from oracle.substrate import available
    if not available():
        pytest.skip("reference substrate not installed")
    from paper_2508_16522_b200.taskbench import generate_graph
    g = generate_graph("stencil_1d", 2, 6, n_workers=2, kind=2, arg=1)
    rows = [g.pred.row(v) for v in range(g.n)]

    def check(it, tok):
        return np.array_equal(tok, seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, np.full(g.n, it, np.uint32), seed=0))

    pts = alg1_cpu.run_sweep(g.n, rows, g.worker, g.kind, [1, 16, 256], processors=2, warmups=0, reps=1,
                             check=check, plateau=0)
    assert [p[0] for p in pts] == [1, 16, 256] and all(p[2] for p in pts) and all(p[1] > 0 for p in pts)
    assert alg1_cpu.compute_peak(1, iters=1 << 10, calls=2, reps=1)["lane_updates_per_s"] > 0
