"""Implicit frontend: dependence analysis KATs (CPU) and the three execution
modes on the GPU."""
import numpy as np
import pytest

from paper_2508_16522_b200.implicit import READ, READWRITE, WRITE, AccessDecl, ImplicitRuntime
from paper_2508_16522_b200.tasks import DeviceBody, TaskRegistry


def _analyze(seq):
    lw, rd, edges = {}, {}, set()
    for i, accs in enumerate(seq):
        for d in ImplicitRuntime.analyze([AccessDecl(r, p) for r, p in accs], lw, rd, i):
            edges.add((d, i))
    return edges


def test_analysis_kat_read_write():
    A, B, C, D = [(0, WRITE)], [(0, READ)], [(0, READ)], [(0, WRITE)]
    assert _analyze([A, B, C, D]) == {(0, 1), (0, 2), (1, 3), (2, 3)}


def test_analysis_two_reads_no_edges():
    assert _analyze([[(0, READ)], [(0, READ)]]) == set()


def test_analysis_waw_single_edge():
    assert _analyze([[(0, WRITE)], [(0, WRITE)]]) == {(0, 1)}


def test_analysis_soundness_and_necessity_random():
    rng = np.random.default_rng(3)
    for _ in range(200):
        n, R = int(rng.integers(1, 30)), int(rng.integers(1, 5))
        seq = [[(int(r), [READ, WRITE, READWRITE][int(rng.integers(0, 3))])
                for r in rng.choice(R, size=int(rng.integers(1, min(R, 2) + 1)), replace=False)] for _ in range(n)]
        E = _analyze(seq)
        reach = [set() for _ in range(n)]
        for j in range(n):
            for i in range(j):
                if (i, j) in E:
                    reach[j] |= reach[i] | {i}
        for j in range(n):
            for i in range(j):
                wi = {r for r, p in seq[i] if p != READ}
                wj = {r for r, p in seq[j] if p != READ}
                ri = {r for r, _ in seq[i]}
                rj = {r for r, _ in seq[j]}
                conflict = bool((wi & rj) | (wj & ri))
                if conflict:
                    assert i in reach[j], (i, j, seq)       # soundness
                if (i, j) in E:
                    assert conflict, (i, j, seq)            # necessity


def _program(rt, regs, n_ops, rng):
    ops = []
    for k in range(n_ops):
        accs = [(int(r), [READ, WRITE, READWRITE][int(rng.integers(0, 3))])
                for r in rng.choice(len(regs), size=int(rng.integers(1, 3)), replace=False)]
        ops.append((1 + k % 3, int(rng.integers(0, 4)), accs))
    return ops


@pytest.mark.gpu
def test_three_modes_identical_memory():
    reg = TaskRegistry()
    reg.register_task(1, DeviceBody.empty())
    reg.register_task(2, DeviceBody.compute_bound(3))
    reg.register_task(3, DeviceBody.busy_wait(100))
    rng = np.random.default_rng(5)
    rt = ImplicitRuntime(reg, seed=9)
    regs = [rt.region() for _ in range(6)]
    prog = _program(rt, regs, 100, rng)
    rt.begin_trace(7)
    for tid, proc, accs in prog:
        rt.issue(tid, proc, accesses=accs)
    rt.end_trace(7)
    untraced = rt.memory_image()
    rt.replay(7, "memoized")
    memo = rt.memory_image()
    done = rt.replay(7, "compiled")
    done.wait()
    comp = rt.memory_image()
    assert untraced == memo == comp and len(comp) > 0
    # re-begin the recorded id -> replay mode, validated against the recording
    rt.begin_trace(7)
    for tid, proc, accs in prog:
        rt.issue(tid, proc, accesses=accs)
    rt.end_trace(7).wait()
    assert rt.memory_image() == comp
    rt.close()


@pytest.mark.gpu
def test_trace_errors():
    from paper_2508_16522_b200.errors import ResourceError, TraceError
    reg = TaskRegistry()
    reg.register_task(1, DeviceBody.empty())
    rt = ImplicitRuntime(reg)
    r = rt.region()
    with pytest.raises(TraceError):
        rt.end_trace(1)
    with pytest.raises(TraceError):
        rt.replay(5, "compiled")
    with pytest.raises(ResourceError):
        rt.issue(1, 0, accesses=[(99, READ)])
    rt.begin_trace(1)
    with pytest.raises(TraceError):
        rt.begin_trace(2)
    rt.issue(1, 0, accesses=[(r, WRITE)])
    rt.end_trace(1)
    rt.begin_trace(1)
    with pytest.raises(TraceError):
        rt.issue(1, 0, accesses=[(r, READ)])
    rt.close()


@pytest.mark.gpu
def test_diamond_trace_two_shards_two_pairs():
    from paper_2508_16522_b200.shard import ShardingPlan
    reg = TaskRegistry()
    for t in (1, 2, 3, 4):
        reg.register_task(t, DeviceBody.empty())
    rt = ImplicitRuntime(reg)
    a, b, c = rt.region(), rt.region(), rt.region()
    rt.begin_trace(3)
    rt.issue(1, 1, accesses=[(a, WRITE)])               # f1 @ P1
    rt.issue(2, 2, accesses=[(a, READ), (b, WRITE)])    # f2 @ P2
    rt.issue(3, 1, accesses=[(a, READ), (c, WRITE)])    # f3 @ P1
    rt.issue(4, 2, accesses=[(b, READ), (c, READ)])     # f4 @ P2
    rt.end_trace(3)
    rt.replay(3, "compiled", ShardingPlan((0, 1), 2)).wait()
    assert rt.ext_pairs(3) == 2
    rt.close()


@pytest.mark.gpu
def test_in_process_multi_gpu_replay():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2508_16522_b200.shard import ShardingPlan
    reg = TaskRegistry()
    for t in (1, 2, 3):
        reg.register_task(t, DeviceBody.compute_bound(t))
    rng = np.random.default_rng(11)
    rt = ImplicitRuntime(reg, seed=4)
    regs = [rt.region() for _ in range(8)]
    prog = _program(rt, regs, 120, rng)
    rt.begin_trace(9)
    for tid, proc, accs in prog:
        rt.issue(tid, proc, accesses=accs)
    rt.end_trace(9)
    untraced = rt.memory_image()
    procs = sorted({p for _, p, _ in prog})
    plan = ShardingPlan(tuple(i % 2 for i in range(len(procs))), 2, devices=(0, 1))
    rt.replay(9, "compiled", plan).wait()
    assert rt.memory_image() == untraced
    assert rt.ext_pairs(9) > 0
    rt.close()


@pytest.mark.gpu
def test_in_process_shards_taskbench():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from oracle import seq
    from paper_2508_16522_b200.shard import InProcessShards, ShardingPlan
    from paper_2508_16522_b200.taskbench import generate_graph
    for pat, W, T in [("stencil_1d", 256, 40), ("all_to_all", 128, 4), ("fft", 128, 20)]:
        g = generate_graph(pat, W, T, n_workers=W)
        sh = InProcessShards(g, ShardingPlan.blocks(W, 2), (0, 1))
        for s in (1, 2):
            sh.run(s)
            np.testing.assert_array_equal(sh.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=s))
        sh.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["memoized", "compiled", "rebegin"])
def test_untraced_ops_after_replay(mode):
    """an untraced op issued after a replay must depend on the
    REPLAYED op that last wrote its region, not on the recording iteration or
    on an untraced writer issued between recording and replay.  The expected
    token is computed with the oracle's token rule (oracle/tokens.py) from the
    replayed op's token and key (its trace-local index)."""
    from oracle import tokens as T
    reg = TaskRegistry()
    reg.register_task(1, DeviceBody.compute_bound(2))
    reg.register_task(2, DeviceBody.empty())
    rt = ImplicitRuntime(reg, seed=13)
    a, b, c = rt.region(), rt.region(), rt.region()
    trace_ops = [(1, 0, [(a, WRITE)]), (1, 1, [(a, READ), (b, WRITE)]), (2, 0, [(b, READ), (a, WRITE)])]
    rt.begin_trace(4)
    for tid, proc, accs in trace_ops:
        rt.issue(tid, proc, accesses=accs)
    rt.end_trace(4)
    u = rt.issue(2, 0, accesses=[(a, WRITE), (b, WRITE)])   # untraced writer between record and replay
    assert u is not None
    if mode == "rebegin":
        rt.begin_trace(4)
        for tid, proc, accs in trace_ops:
            rt.issue(tid, proc, accesses=accs)
        rt.end_trace(4).wait()
    else:
        done = rt.replay(4, mode)
        if done is not None:
            done.wait()
    # trace tokens after the replay: op 2 last wrote a, op 1 last wrote b
    img = rt.memory_image()
    ta, tb = img[a], img[b]
    seq_x = rt._seq
    x = rt.issue(1, 0, accesses=[(a, READ), (b, READ), (c, WRITE)])
    assert x is not None
    got = rt.memory_image()[c]
    want = T.token_int(13, seq_x, sorted([(2, ta), (1, tb)]), T.BODY_COMPUTE, 2)
    assert got == want
    rt.close()
