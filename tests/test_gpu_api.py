"""GPU: the SPEC-level public API through the C ABI — compile/execute with
external pre/postconditions, message_stats, error conventions, timeouts."""
import threading
import time

import numpy as np
import pytest

from oracle import seq
from paper_2508_16522_b200 import _native as N
from paper_2508_16522_b200.compiler import Event, compile as td_compile
from paper_2508_16522_b200.errors import CompileError, ExecutionStateError, WaitTimeout
from paper_2508_16522_b200.graph import ExtPostcond, ExtPrecond, Task, build
from paper_2508_16522_b200.tasks import DeviceBody, TaskRegistry

pytestmark = pytest.mark.gpu


def _reg():
    r = TaskRegistry()
    r.register_task(1, DeviceBody.empty())
    r.register_task(2, DeviceBody.compute_bound(5))
    r.register_task(3, DeviceBody.busy_wait(2000))
    r.register_task(4, DeviceBody.empty())
    return r


def _oracle_tokens(g, seed):
    kind = np.array(g.flat.kind)
    kind[(kind == 4) | (kind == 5)] = 0   # ext nodes carry no body
    return seq.run_c(g.flat.n, g.flat.pred.ptr, g.flat.pred.iv, kind, g.flat.arg, seed=seed,
                     order=np.argsort(g.flat.order))


def test_diamond_message_stats():
    g = build([Task(1, 1), Task(2, 2), Task(1, 1), Task(2, 4)], [(0, 1), (0, 2), (1, 3), (2, 3)])
    cg = td_compile(g, registry=_reg())
    done, post = cg.execute(seed=3)
    done.wait()
    assert cg.message_stats() == dict(cross_worker_messages=2, local_decrements=2, init_messages=2)
    np.testing.assert_array_equal(cg.tokens(), _oracle_tokens(cg, 3))
    cg.close()


def test_external_pre_and_post_conditions():
    nodes = [ExtPrecond(0), Task(0, 2), Task(1, 3), Task(0, 1), ExtPostcond(0), ExtPrecond(1), Task(1, 2)]
    edges = [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4), (5, 6), (6, 4)]
    g = build(nodes, edges)
    cg = td_compile(g, registry=_reg())
    gate = threading.Event()
    pre0 = Event(gate.is_set)               # pending host event
    done, post = cg.execute([pre0, Event.triggered()], seed=7)
    time.sleep(0.05)
    assert not done.query() and not post[0].query()   # blocked on precondition 0
    gate.set()
    done.wait(10)
    assert post[0].query()
    np.testing.assert_array_equal(cg.tokens(), _oracle_tokens(cg, 7))
    cg.close()


def test_never_triggered_precondition_times_out_then_recovers():
    g = build([ExtPrecond(0), Task(0, 1), Task(0, 2)], [(0, 1), (1, 2)])
    cg = td_compile(g, registry=_reg())
    done, _ = cg.execute([Event(lambda: False)], seed=1)
    with pytest.raises(WaitTimeout):
        done.wait(0.2)
    done, _ = cg.execute([Event.triggered()], seed=1)   # the graph stays usable
    done.wait(10)
    np.testing.assert_array_equal(cg.tokens(), _oracle_tokens(cg, 1))
    cg.close()


def test_outstanding_execution_rejected():
    g = build([ExtPrecond(0), Task(0, 1)], [(0, 1)])
    cg = td_compile(g, registry=_reg())
    gate = threading.Event()
    done, _ = cg.execute([Event(gate.is_set)])
    with pytest.raises(ExecutionStateError):
        cg.execute([Event.triggered()])
    gate.set()
    done.wait(10)
    cg.execute([Event.triggered()])[0].wait(10)
    cg.close()


def test_compile_errors():
    reg = _reg()
    reg.register_task(9, lambda rt, args: None)   # host-only body
    with pytest.raises(CompileError):
        td_compile(build([Task(0, 77)], []), registry=reg)
    with pytest.raises(CompileError):
        td_compile(build([Task(0, 9)], []), registry=reg)


def test_empty_graph_and_single_node():
    cg = td_compile(build([], []), registry=_reg())
    cg.execute()[0].wait(10)
    cg.close()
    cg = td_compile(build([Task(3, 2)], []), registry=_reg())
    cg.execute(seed=4)[0].wait(10)
    assert cg.message_stats()["cross_worker_messages"] == 0
    np.testing.assert_array_equal(cg.tokens(), _oracle_tokens(cg, 4))
    cg.close()


def test_spin_limit_poisons():  # SPEC.md:383 poisoned marker
    from paper_2508_16522_b200.errors import ExecutionPoisoned
    g = build([ExtPrecond(0), Task(0, 1), Task(1, 1)], [(0, 1), (1, 2)])
    cg = td_compile(g, registry=_reg())
    done, _ = cg.execute([Event(lambda: False)], spin_limit=1 << 14)
    with pytest.raises((ExecutionPoisoned, WaitTimeout)):
        done.wait(5)
    cg.execute([Event.triggered()])[0].wait(10)
    np.testing.assert_array_equal(cg.tokens(), _oracle_tokens(cg, 0))
    cg.close()


def test_mailbox_indegree_limit():
    """a node with 65,536 in-edges overflows the 16-bit count field of its
    mailbox word: rejected at compile (upload) time, not silently wrong"""
    from paper_2508_16522_b200.errors import CompileError
    from paper_2508_16522_b200.executor import DeviceGraph
    from paper_2508_16522_b200.taskbench import generate_graph
    g = generate_graph("all_to_all", 65536, 2, n_workers=1024)
    with pytest.raises(CompileError):
        DeviceGraph(g)
    g = generate_graph("all_to_all", 65535, 2, n_workers=1024)   # the largest legal fan-in
    with DeviceGraph(g) as dg:
        dg.run(seed=2)
        from oracle import seq
        np.testing.assert_array_equal(dg.tokens(), seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=2))


def test_poison_is_sticky_across_queued_launches():
    """a queued (TD_F_QUEUE) launch behind a poisoned execution
    must not clear the poison: waiting reports the FIRST failure, and the
    next un-queued launch (after the dirty-graph memset) is correct again."""
    from paper_2508_16522_b200.errors import ExecutionPoisoned
    g = build([ExtPrecond(0), Task(0, 1), Task(1, 1)], [(0, 1), (1, 2)])
    cg = td_compile(g, registry=_reg())
    dev = cg.dev
    dev.launch(0, flags=0, spin_limit=1 << 14)            # precondition never triggered: poisons
    dev.launch(0, flags=N.TD_F_QUEUE, spin_limit=0)        # queued behind it
    with pytest.raises(ExecutionPoisoned, match="spin limit"):
        dev.wait(20)
    dev.trigger_pre(0)
    dev.launch(3, flags=0)
    dev.trigger_pre(0)
    dev.wait(20)
    np.testing.assert_array_equal(dev.tokens(), _oracle_tokens(cg, 3))
    cg.close()
