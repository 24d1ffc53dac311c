"""CPU: graph file format round trips and the .npz
form of recorded traces."""
import numpy as np
import pytest

from paper_2508_16522_b200.errors import GraphError, GraphParseError
from paper_2508_16522_b200.flat import load_npz, save_npz
from paper_2508_16522_b200.graph import Copy, ExtPostcond, ExtPrecond, Task, build, from_json, to_json
from paper_2508_16522_b200.taskbench import generate_graph

DIAMOND = build([Task(1, 1, b"\x01"), Task(2, 2), Task(1, 3), Task(2, 4)], [(0, 1), (0, 2), (1, 3), (2, 3)])


def test_diamond_roundtrip():
    g2 = from_json(to_json(DIAMOND))
    assert g2.nodes == DIAMOND.nodes and g2.edges == DIAMOND.edges


def test_ext_and_copy_roundtrip():
    g = build([ExtPrecond(0), Task(0, 7), Copy(0, 1, 64), ExtPostcond(0)], [(0, 1), (1, 2), (2, 3)])
    g2 = from_json(to_json(g))
    assert g2.nodes == g.nodes and g2.edges == g.edges
    assert (g2.n_ext_pre, g2.n_ext_post) == (1, 1)


def test_malformed_text_parse_error_with_position():
    with pytest.raises(GraphParseError) as e:
        from_json('{"version": 1,\n "nodes": [}')
    assert e.value.line == 2


def test_cyclic_file_rejected():
    import json
    doc = json.loads(to_json(DIAMOND))
    doc["edges"].append({"src": 3, "dst": 0, "kind": "host"})
    with pytest.raises(GraphError):
        from_json(json.dumps(doc))


@pytest.mark.parametrize("pat", ["stencil_1d", "fft", "all_to_all", "tree"])
def test_flat_npz_roundtrip(tmp_path, pat):
    g = generate_graph(pat, 64, 20, n_workers=16)
    p = str(tmp_path / "t.npz")
    save_npz(g, p)
    h = load_npz(p)
    for a, b in [(g.pred.ptr, h.pred.ptr), (g.pred.iv, h.pred.iv), (g.succ.ptr, h.succ.ptr),
                 (g.succ.iv, h.succ.iv), (g.kind, h.kind), (g.arg, h.arg), (g.worker, h.worker), (g.col, h.col)]:
        assert np.array_equal(a, b)
    assert h.n == g.n and h.n_workers == g.n_workers and h.meta["pattern"] == g.meta["pattern"]


def test_transitive_reduce_kats():
    from paper_2508_16522_b200.graph import transitive_reduce
    g = build(list(DIAMOND.nodes), list(DIAMOND.edges) + [(0, 3)])
    assert transitive_reduce(g).edges == DIAMOND.edges          # (f1,f4) removed
    assert transitive_reduce(DIAMOND).edges == DIAMOND.edges    # already reduced
    assert transitive_reduce(build([], [])).edges == ()


def test_transitive_reduce_random_dags():
    from paper_2508_16522_b200.graph import reachability, transitive_reduce
    rng = np.random.default_rng(7)
    for _ in range(150):
        n = int(rng.integers(1, 65))
        e = set()
        for v in range(1, n):
            for u in rng.choice(v, size=int(rng.integers(0, min(v, 6) + 1)), replace=False):
                e.add((int(u), v))
        g = build([Task(0, 1)] * n, sorted(e))
        r = transitive_reduce(g)
        assert np.array_equal(reachability(g), reachability(r))
        # minimal: removing any remaining edge changes reachability
        R = reachability(r)
        for (a, b) in r.edges:
            alt = any(R[s, b] for s in r.succ.row(a) if s != b)
            assert not alt
