"""Host-task interop on the GPU (§4.3): an
async-transformed graph runs its host nodes on the CPU and its device work in
the persistent kernel; a host node waits only for device work it consumes
(sync edges), and device work starts when its host side issued it."""
import numpy as np
import pytest

from paper_2508_16522_b200.graph import Task, async_transform, build
from paper_2508_16522_b200.hybrid import HybridGraph
from paper_2508_16522_b200.tasks import DeviceBody, TaskRegistry

pytestmark = pytest.mark.gpu


def test_hybrid_run_ahead_and_sync():
    reg = TaskRegistry()
    seen = {}
    hg = None

    def host(tag):
        def f(_args):
            a_post = hg.post_of[hg_async_of[0]]
            seen[tag] = hg.cg.dev.post_fired(a_post)
        return f

    reg.register_task(1, DeviceBody.busy_wait(20_000_000))  # A: 20 ms of device work
    reg.register_task(2, host("X"))                          # X: host only, independent of A's device work
    reg.register_task(3, host("B"))                          # B: consumes A's device work (sync edge)
    reg.register_task(4, DeviceBody.compute_bound(7))        # C: device work after B
    reg.register_task(5, lambda _a: None)                    # H0: host root
    # H0 -> A(dev) -> B(host) -> C(dev); H0 -> X(host)
    g = build([Task(0, 5), Task(0, 1, device_work=True), Task(0, 2), Task(0, 3), Task(1, 4, device_work=True)],
              [(0, 1), (0, 2), (1, 3), (3, 4)])
    t = async_transform(g)
    hg = HybridGraph(t, registry=reg)
    hg_async_of = {t.nodes[v].of: v for v in hg.async_nodes}
    hg_async_of[0] = hg_async_of[1]
    try:
        for seed in (1, 2):
            seen.clear()
            hg.execute(seed=seed)
            assert seen["X"] is False     # ran ahead of A's 3 ms of device work
            assert seen["B"] is True      # waited for it
            order = [v for v, _ in hg.host_log]
            assert order.index(3) > order.index(0)
            # device tokens: the device graph replayed bit-exactly
            from oracle import seq
            f = hg.cg.flat
            kind = np.array(f.kind)
            kind[(kind == 4) | (kind == 5)] = 0   # ext nodes carry no body
            want = seq.run_c(f.n, f.pred.ptr, f.pred.iv, kind, f.arg, seed=seed, order=np.argsort(f.order))
            np.testing.assert_array_equal(hg.tokens(), want)
    finally:
        hg.close()


def test_hybrid_all_device_chain():
    reg = TaskRegistry()
    reg.register_task(1, DeviceBody.compute_bound(3))
    g = build([Task(0, 1, device_work=True) for _ in range(6)], [(i, i + 1) for i in range(5)])
    hg = HybridGraph(async_transform(g), registry=reg)
    try:
        hg.execute(seed=9)
        assert len(hg.post_of) == 0          # no sync edges: everything stays on the device
        assert hg.device_graph.n == 12       # 6 async nodes + 6 launch preconditions
    finally:
        hg.close()
