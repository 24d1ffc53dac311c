"""ctypes binding of libtdexec.so (include/tdexec.h) and its nvcc build.

There is no CPU fallback: if the shared library is missing or fails to load,
every executor entry point raises.  ``build()`` compiles it in-tree for
sm_100a (``nvcc -gencode arch=compute_100a,code=sm_100a``) so the .so travels
with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

from .errors import DeviceError, raise_for_status

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libtdexec.so")
SRC_PATH = os.path.join(PKG_DIR, "csrc", "tdexec.cu")
MB_LIB_PATH = os.path.join(PKG_DIR, "libtdmicro.so")
MB_SRC_PATH = os.path.join(PKG_DIR, "csrc", "microbench.cu")
CMP_LIB_PATH = os.path.join(PKG_DIR, "libtdcmp.so")
CMP_SRC_PATH = os.path.join(PKG_DIR, "csrc", "comparators.cu")
HDR_PATH = os.path.join(REPO_DIR, "include", "tdexec.h")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-shared", "-std=c++17", "-lgomp"]

# body kinds / flags (tdexec.h)
(TD_BODY_EMPTY, TD_BODY_BUSY_WAIT, TD_BODY_COMPUTE, TD_BODY_STENCIL2D, TD_BODY_EXT_PRE, TD_BODY_EXT_POST,
 TD_BODY_MEMORY) = range(7)
TD_F_CHECKSUM, TD_F_STATS, TD_F_TALLY, TD_F_QUEUE, TD_F_TRACE, TD_F_DYNAMIC = 1, 2, 4, 8, 16, 32
TD_UPLOAD_DYNAMIC = 1


class TdCsr(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("pred_ptr", C.c_void_p), ("pred_iv", C.c_void_p),
        ("succ_ptr", C.c_void_p), ("succ_iv", C.c_void_p),
        ("kind", C.c_void_p), ("arg", C.c_void_p),
        ("n_workers", C.c_int32), ("work_ptr", C.c_void_p), ("work", C.c_void_p),
        ("n_cols", C.c_int32), ("col", C.c_void_p),
        ("n_ranks", C.c_int32), ("my_rank", C.c_int32), ("node_rank", C.c_void_p),
        ("n_ext_pre", C.c_int32), ("n_ext_post", C.c_int32),
        ("ident", C.c_void_p),
        ("options", C.c_uint32),
    ]


class TdLaunchParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("flags", C.c_uint32),
                ("threads_per_block", C.c_uint32), ("spin_limit", C.c_uint64)]


class TdStats(C.Structure):
    _fields_ = [
        ("executed", C.c_uint64), ("cross_worker_edges", C.c_uint64),
        ("local_decrements", C.c_uint64), ("init_messages", C.c_uint64),
        ("cross_rank_edges", C.c_uint64), ("epoch", C.c_uint64),
        ("poisoned", C.c_int32), ("workers", C.c_int32), ("blocks", C.c_int32),
        ("threads_per_block", C.c_int32),
    ]


class TdDeviceInfo(C.Structure):
    _fields_ = [("sm_count", C.c_int32), ("l2_bytes", C.c_int32), ("max_workers", C.c_int32),
                ("max_workers_st2d", C.c_int32),
                ("cc_major", C.c_int32), ("cc_minor", C.c_int32), ("name", C.c_char * 96)]


class TdGraphInfo(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_positions", C.c_int64), ("n_shared", C.c_int64),
                ("n_workers", C.c_int32), ("n_graph_workers", C.c_int32),
                ("n_ranks", C.c_int32), ("my_rank", C.c_int32), ("plain", C.c_int32), ("group", C.c_int32),
                ("has_stencil2d", C.c_int32), ("desc_bytes", C.c_int32), ("slot_shift", C.c_int32),
                ("n_combiners", C.c_int32)]


EXPORTED = (
    "td_last_error", "td_device_info_get", "td_graph_upload", "td_graph_launch",
    "td_graph_wait", "td_graph_query", "td_graph_trigger_pre", "td_graph_post_fired",
    "td_graph_tokens", "td_graph_checksums", "td_graph_tally", "td_graph_stats",
    "td_graph_last_ms", "td_graph_trace", "td_graph_ipc_export", "td_graph_ipc_attach", "td_graph_peer_attach_direct", "td_graph_destroy",
    "td_graph_attach_stencil2d", "td_graph_stencil2d_grid", "td_graph_set_body_arg", "td_graph_info_get",
    "td_graph_attach_scratch",
    "td_rt_create", "td_rt_launch_task", "td_rt_store_tokens", "td_rt_sync", "td_rt_tokens", "td_rt_destroy",
)

_lib = None
_lock = threading.Lock()


def _nvcc(src: str, out: str, deps: list[str], force: bool, verbose: bool) -> str:
    if not force and os.path.exists(out):
        if os.path.getmtime(out) >= max(os.path.getmtime(d) for d in [src, *deps]):
            return out
    cmd = ["nvcc", *NVCC_FLAGS, "-o", out + ".tmp", src]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True, cwd=os.path.dirname(src))
    os.replace(out + ".tmp", out)
    return out


def build(force: bool = False, verbose: bool = False) -> list[str]:
    """Compile the executor (csrc/tdexec.cu -> libtdexec.so) and the K3
    microbenchmarks (csrc/microbench.cu -> libtdmicro.so) for sm_100a, in-tree."""
    return [_nvcc(SRC_PATH, LIB_PATH, [HDR_PATH], force, verbose),
            _nvcc(MB_SRC_PATH, MB_LIB_PATH, [], force, verbose),
            _nvcc(CMP_SRC_PATH, CMP_LIB_PATH, [], force, verbose)]


def lib():
    """Load libtdexec.so (raises if absent: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("TD_LIB") or LIB_PATH  # TD_LIB: a diagnostic build of the same source
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                "The executor has no CPU fallback.")
        L = C.CDLL(path)
        vp, i32, i64, u32, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
        L.td_last_error.restype = C.c_char_p
        L.td_last_error.argtypes = []
        sig = {
            "td_device_info_get": [i32, u32, C.POINTER(TdDeviceInfo)],
            "td_graph_upload": [C.POINTER(TdCsr), i32, C.POINTER(vp)],
            "td_graph_launch": [vp, C.POINTER(TdLaunchParams), vp],
            "td_graph_wait": [vp, dbl],
            "td_graph_query": [vp, C.POINTER(i32)],
            "td_graph_trigger_pre": [vp, i32],
            "td_graph_post_fired": [vp, i32, C.POINTER(i32)],
            "td_graph_tokens": [vp, vp, i64],
            "td_graph_checksums": [vp, vp, i32],
            "td_graph_tally": [vp, vp, i64],
            "td_graph_stats": [vp, C.POINTER(TdStats)],
            "td_graph_last_ms": [vp, C.POINTER(C.c_float)],
            "td_graph_info_get": [vp, C.POINTER(TdGraphInfo)],
            "td_graph_attach_scratch": [vp, i64],
            "td_graph_trace": [vp, vp, i64],
            "td_graph_ipc_export": [vp, vp, C.c_size_t, C.POINTER(C.c_size_t)],
            "td_graph_ipc_attach": [vp, i32, vp, C.c_size_t],
            "td_graph_peer_attach_direct": [vp, i32, vp],
            "td_graph_destroy": [vp],
            "td_graph_attach_stencil2d": [vp, i32, i32],
            "td_graph_set_body_arg": [vp, u32],
            "td_graph_stencil2d_grid": [vp, i32, vp, i64],
            "td_rt_create": [i32, i64, C.POINTER(vp)],
            "td_rt_launch_task": [vp, i64, C.c_uint64, C.c_uint8, u32, C.c_uint64, vp, i32],
            "td_rt_store_tokens": [vp, vp, vp, vp, i32],
            "td_rt_sync": [vp],
            "td_rt_tokens": [vp, i64, i64, vp],
            "td_rt_destroy": [vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.restype = i32
            f.argtypes = args
        _lib = L
        return _lib


def check(status: int) -> None:
    if status:
        msg = lib().td_last_error().decode(errors="replace")
        raise_for_status(status, msg)
