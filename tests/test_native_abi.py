"""CPU: the C-ABI library loads and exports every symbol include/tdexec.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

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


def _header_struct_fields(name):
    """Field names of `typedef struct name { ... } name;` in include/tdexec.h, in order."""
    src = open(HDR).read()
    m = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), src, re.S)
    assert m, name
    body = re.sub(r"/\*.*?\*/", "", m.group(1), flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        # "int32_t n_ranks, my_rank" / "const int64_t* pred_ptr" / "uint32_t options"
        names = [re.sub(r"\[.*\]", "", p).strip().lstrip("*").strip() for p in decl.split(",")]
        names[0] = names[0].split()[-1].lstrip("*")
        fields += names
    return fields


@pytest.mark.parametrize("cname,pyname", [("td_csr", "TdCsr"), ("td_launch_params", "TdLaunchParams"),
                                          ("td_stats", "TdStats"), ("td_device_info", "TdDeviceInfo"),
                                          ("td_graph_info", "TdGraphInfo")])
def test_ctypes_structs_match_the_header(cname, pyname):
    """The ctypes mirrors in _native.py list the header's fields in the header's order
    (a field added to one side only would silently shift every later field)."""
    want = _header_struct_fields(cname)
    got = [f for f, _ in getattr(N, pyname)._fields_]
    assert got == want, (cname, want, got)


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the shared library absent the binding raises instead
    of running anything (checked in a subprocess with TD_LIB pointing nowhere)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2508_16522_b200 import _native as N\n"
            "from paper_2508_16522_b200.errors import DeviceError\n"
            "try:\n    N.lib()\nexcept DeviceError as e:\n    print('raised', 'no CPU fallback' in str(e))\n"
            "else:\n    print('loaded')\n") % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TD_LIB=str(tmp_path / "absent.so"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert out.stdout.strip() == "raised True", out.stdout + out.stderr
