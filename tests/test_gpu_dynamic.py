"""GPU: the arrival-order (per-SM ready queue) dispatch mode, TD_F_DYNAMIC
(a node is dispatched the moment its counter hits zero),
bit-exact against the oracle and exactly-once, interchangeable with the
static-list mode on the same upload."""
import numpy as np
import pytest

from paper_2508_16522_b200 import _native as N
from paper_2508_16522_b200.executor import DeviceGraph
from paper_2508_16522_b200.flat import FlatGraph, IntervalCSR, transpose
from paper_2508_16522_b200.taskbench import generate_graph
from oracle import seq

pytestmark = pytest.mark.gpu


def _oracle(g, seed):
    return seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=seed)


@pytest.mark.parametrize("pattern,W,T,workers,kind,arg", [
    ("stencil_1d", 64, 30, 64, 2, 3), ("stencil_1d", 1024, 100, 128, 2, 1), ("no_comm", 200, 10, 50, 0, 0),
    ("fft", 256, 20, 64, 2, 2), ("tree", 512, 12, 32, 0, 0), ("nearest", 300, 8, 300, 0, 0),
    ("all_to_all", 200, 4, 40, 0, 0), ("spread", 64, 10, 16, 1, 200), ("stencil_1d", 8, 100, 8, 0, 0)])
def test_dynamic_matches_oracle(pattern, W, T, workers, kind, arg):
    g = generate_graph(pattern, W, T, n_workers=workers, mapping="block", kind=kind, arg=arg)
    with DeviceGraph(g, dynamic=True) as dg:
        for seed, flags in ((1, N.TD_F_DYNAMIC | N.TD_F_TALLY | N.TD_F_STATS), (2, N.TD_F_DYNAMIC | N.TD_F_CHECKSUM),
                            (3, 0), (4, N.TD_F_DYNAMIC)):   # static and dynamic launches interleaved
            dg.run(seed=seed, flags=flags, spin_limit=1 << 24)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, seed))
            if flags & N.TD_F_TALLY:
                assert (dg.tally() == 1).all()
                assert dg.stats()["executed"] == g.n


def test_dynamic_random_dags():
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 200))
        rows = []
        for v in range(n):
            k = int(rng.integers(0, min(v, 7) + 1)) if v else 0
            rows.append(sorted(rng.choice(v, size=k, replace=False).tolist()) if k else [])
        pred = IntervalCSR.from_lists(n, rows)
        P = int(rng.integers(1, 9))
        g = FlatGraph(n=n, pred=pred, succ=transpose(pred), kind=rng.choice([0, 1, 2], size=n).astype(np.uint8),
                      arg=rng.integers(0, 50, size=n).astype(np.uint32),
                      worker=rng.integers(0, P, size=n).astype(np.int32), n_workers=P)
        want = np.array(seq.run_py(n, rows, g.kind, g.arg, seed=trial), dtype=np.uint64)
        with DeviceGraph(g, dynamic=True) as dg:
            dg.run(seed=trial, flags=N.TD_F_DYNAMIC | N.TD_F_TALLY, spin_limit=1 << 24)
            np.testing.assert_array_equal(dg.tokens(), want)
            assert (dg.tally() == 1).all()


def test_dynamic_memory_bound_and_errors():
    from paper_2508_16522_b200.errors import ContractViolation
    g = generate_graph("stencil_1d", 64, 10, n_workers=16, mapping="block", kind=6, arg=128)
    with DeviceGraph(g, dynamic=True) as dg:
        dg.attach_scratch(128)
        dg.run(seed=5, flags=N.TD_F_DYNAMIC, spin_limit=1 << 24)
        np.testing.assert_array_equal(dg.tokens(), _oracle(g, 5))
    g = generate_graph("stencil_1d", 16, 4)
    with DeviceGraph(g) as dg:                      # uploaded without the dynamic programs
        with pytest.raises(ContractViolation):
            dg.run(seed=1, flags=N.TD_F_DYNAMIC)


def test_dynamic_imbalanced_busy_wait():
    """Variable-length bodies on multi-column workers: the case arrival-order
    dispatch is for (a ready node is never stuck behind an unready list head)."""
    rng = np.random.default_rng(3)
    g = generate_graph("stencil_1d", 256, 40, n_workers=32, mapping="block", kind=1, arg=0)
    g.arg[:] = rng.integers(0, 3000, size=g.n).astype(np.uint32)
    with DeviceGraph(g, dynamic=True) as dg:
        for flags in (N.TD_F_DYNAMIC, 0):
            dg.run(seed=8, flags=flags, spin_limit=1 << 24)
            np.testing.assert_array_equal(dg.tokens(), _oracle(g, 8))


def test_dynamic_large_ids():
    """More than 2^16 nodes: queue-slot tags wrap (id mod 65535 + 1)."""
    g = generate_graph("stencil_1d", 1024, 80, n_workers=200, mapping="block", kind=0, arg=0)
    with DeviceGraph(g, dynamic=True) as dg:
        dg.run(seed=2, flags=N.TD_F_DYNAMIC | N.TD_F_TALLY, spin_limit=1 << 24)
        np.testing.assert_array_equal(dg.tokens(), _oracle(g, 2))
        assert (dg.tally() == 1).all()
