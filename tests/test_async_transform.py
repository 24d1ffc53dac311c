"""async_transform (§4.3, Fig. 9) and the edge-kind
aware graph formats -- CPU known-answer tests from the SPEC's examples."""
import pytest

from paper_2508_16522_b200.errors import CompileError
from paper_2508_16522_b200.graph import (AsyncNode, Task, async_transform, build, from_json, to_dot, to_json,
                                         transitive_reduce)


def _edges(g):
    return {e: g.edge_kind(i) for i, e in enumerate(g.edges)}


def test_chain_all_device_work():
    """n1->n2->n3, all with device work: n1a, n2a, n3a and async edges
    (n1a,n2a), (n2a,n3a); no sync edges"""
    g = build([Task(0, 1, device_work=True), Task(0, 2, device_work=True), Task(0, 3, device_work=True)],
              [(0, 1), (1, 2)])
    t = async_transform(g)
    assert t.nodes[3:] == (AsyncNode(0), AsyncNode(1), AsyncNode(2))
    e = _edges(t)
    assert {k for k, v in e.items() if v == "async"} == {(3, 4), (4, 5)}
    assert not [k for k, v in e.items() if v == "sync"]
    assert {k for k, v in e.items() if v == "host"} == {(0, 1), (1, 2)}       # host edges retained
    assert {k for k, v in e.items() if v == "launch"} == {(0, 3), (1, 4), (2, 5)}


def test_chain_partial_device_work():
    """n1->n2, only n1 has device work: sync edge (n1a, n2)"""
    t = async_transform(build([Task(0, 1, device_work=True), Task(0, 2)], [(0, 1)]))
    assert t.nodes[2] == AsyncNode(0)
    assert _edges(t) == {(0, 1): "host", (0, 2): "launch", (2, 1): "sync"}


def test_no_device_work_is_identity():
    g = build([Task(0, 1), Task(1, 2)], [(0, 1)])
    assert async_transform(g) is g


def test_diamond_mixed():
    # f1(dev) -> f2(host), f1 -> f3(dev), f2 -> f4(dev), f3 -> f4
    g = build([Task(1, 1, device_work=True), Task(2, 2), Task(1, 3, device_work=True),
               Task(2, 4, device_work=True)], [(0, 1), (0, 2), (1, 3), (2, 3)])
    t = async_transform(g)
    a = {x.of: v for v, x in enumerate(t.nodes) if isinstance(x, AsyncNode)}
    e = _edges(t)
    assert e[(a[0], 1)] == "sync" and e[(a[0], a[2])] == "async" and e[(a[2], a[3])] == "async"
    assert (1, a[3]) not in e            # f2 has no device work: nothing leaves it but its host edge
    assert len(t.nodes) == 7


def test_formats_keep_edge_kinds():
    t = async_transform(build([Task(0, 1, device_work=True), Task(0, 2)], [(0, 1)]))
    assert from_json(to_json(t)) == t
    assert _edges(from_json(to_json(t))) == _edges(t)
    dot = to_dot(t)
    assert "style=dashed" in dot and 'label="sync"' in dot and dot.count("->") == 3
    r = _edges(transitive_reduce(t))      # (0,1) is implied by launch + sync: dropped
    assert r == {k: v for k, v in _edges(t).items() if k != (0, 1)}


def test_compile_refuses_async_graphs():
    from paper_2508_16522_b200.compiler import compile as td_compile
    t = async_transform(build([Task(0, 1, device_work=True), Task(0, 2)], [(0, 1)]))
    with pytest.raises(CompileError):
        td_compile(t)
