"""CPU: the C-ABI library loads and exports every symbol include/tdexec.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from paper_2508_16522_b200 import _native as N

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "tdexec.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:td_status|const char\*)\s+(td_\w+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    d = declared()
    assert "td_graph_upload" in d and "td_graph_launch" in d and "td_graph_wait" in d
    assert set(d) == set(N.EXPORTED)


def test_library_exports_every_declared_symbol():
    N.build()
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name


def test_binding_loads():
    L = N.lib()
    assert L.td_last_error() is not None


def test_status_codes_map_to_reference_errors():
    from paper_2508_16522_b200 import errors as E
    src = open(HDR).read()
    codes = dict((m, int(c)) for m, c in re.findall(r"(TD_E_\w+)\s*=\s*(\d+)", src))
    assert E.STATUS_CLASSES[codes["TD_E_EXEC_STATE"]] is E.ExecutionStateError
    assert E.STATUS_CLASSES[codes["TD_E_GRAPH"]] is E.GraphError
    assert E.STATUS_CLASSES[codes["TD_E_COMPILE"]] is E.CompileError
    assert E.STATUS_CLASSES[codes["TD_E_WAIT_TIMEOUT"]] is E.WaitTimeout
    assert E.STATUS_CLASSES[codes["TD_E_POISONED"]] is E.ExecutionPoisoned
