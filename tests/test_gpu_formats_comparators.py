"""GPU: replaying persisted traces (the on-disk
graph format, .npz and the SPEC JSON form) and the paper's comparators
(the same DAG as a CUDA Graph and through a generic
per-task event runtime), each bit-exact against the oracle."""
import os

import numpy as np
import pytest

from paper_2508_16522_b200 import _native as N
from paper_2508_16522_b200.comparators import CudaGraphReplay, event_runtime
from paper_2508_16522_b200.executor import DeviceGraph
from paper_2508_16522_b200.flat import load_npz, save_npz
from paper_2508_16522_b200.implicit import READ, WRITE, ImplicitRuntime
from paper_2508_16522_b200.tasks import DeviceBody, TaskRegistry
from paper_2508_16522_b200.taskbench import generate_graph
from oracle import seq

pytestmark = pytest.mark.gpu


def _oracle(g, seed):
    order = None if g.order is None else np.argsort(g.order)
    return seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=seed, order=order)


def test_recorded_trace_saved_loaded_replayed(tmp_path):
    """record -> save_trace(.npz) -> load_npz -> upload -> replay: the loaded
    graph gives the same tokens as the in-memory compiled replay and the
    oracle."""
    reg = TaskRegistry()
    reg.register_task(1, DeviceBody.compute_bound(5))
    reg.register_task(2, DeviceBody.empty())
    rt = ImplicitRuntime(reg, seed=21)
    regs = [rt.region() for _ in range(5)]
    rng = np.random.default_rng(2)
    rt.begin_trace(1)
    for k in range(80):
        accs = [(regs[int(r)], [READ, WRITE][int(rng.integers(0, 2))])
                for r in rng.choice(5, size=int(rng.integers(1, 3)), replace=False)]
        rt.issue(1 + k % 2, int(rng.integers(0, 3)), accesses=accs)
    rt.end_trace(1)
    rt.replay(1, "compiled").wait()
    live = rt._traces[1].compiled.tokens()
    path = os.path.join(tmp_path, "trace.npz")
    rt.save_trace(1, path)
    g = load_npz(path)
    with DeviceGraph(g) as dg:
        dg.run(seed=21)
        np.testing.assert_array_equal(dg.tokens(), live[:g.n])
        np.testing.assert_array_equal(dg.tokens(), _oracle(g, 21))
    rt.close()


@pytest.mark.parametrize("pattern,W,T", [("stencil_1d", 64, 40), ("fft", 128, 12), ("all_to_all", 64, 4)])
def test_taskbench_graph_npz_round_trip_replay(pattern, W, T, tmp_path):
    g = generate_graph(pattern, W, T, kind=2, arg=2)
    p = os.path.join(tmp_path, "g.npz")
    save_npz(g, p)
    g2 = load_npz(p)
    with DeviceGraph(g2) as dg:
        dg.run(seed=6, flags=N.TD_F_CHECKSUM)
        np.testing.assert_array_equal(dg.tokens(), _oracle(g, 6))


@pytest.mark.parametrize("pattern,W,T", [("stencil_1d", 8, 30), ("fft", 32, 12), ("nearest", 24, 10)])
def test_comparators_bit_exact(pattern, W, T):
    g = generate_graph(pattern, W, T, n_workers=W, kind=2, arg=3)
    want = _oracle(g, 4)
    cg = CudaGraphReplay(g, seed=4)
    cg.run()
    np.testing.assert_array_equal(cg.tokens(), want)
    assert cg.run() > 0
    cg.close()
    ms, tok = event_runtime(g, min(W, 16), seed=4)
    assert ms > 0
    np.testing.assert_array_equal(tok, want)


def test_spec_json_graph_round_trip_replay():
    """A TaskGraph written in the SPEC file format and read
    back compiles and replays to the same tokens as the original."""
    from paper_2508_16522_b200.compiler import compile as td_compile
    from paper_2508_16522_b200.graph import Task, build, from_json, to_json
    reg = TaskRegistry()
    reg.register_task(1, DeviceBody.compute_bound(4))
    reg.register_task(2, DeviceBody.empty())
    rng = np.random.default_rng(4)
    n = 120
    edges = sorted({(int(u), v) for v in range(1, n) for u in rng.choice(v, size=min(v, 3), replace=False)})
    g = build([Task(i % 5, 1 + (i % 2)) for i in range(n)], edges)
    g2 = from_json(to_json(g))
    toks = []
    for gg in (g, g2):
        cg = td_compile(gg, registry=reg)
        cg.execute(seed=8)[0].wait(30)
        toks.append(cg.tokens())
        cg.close()
    np.testing.assert_array_equal(toks[0], toks[1])
