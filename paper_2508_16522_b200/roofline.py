"""K3 roofline microbenchmarks (§8(d)).

Measures, on the box, the denominators of
    R_roof = min(A_L2 / atomics_task, BW / bytes_task, W_active / L_level)
and writes them as a dict (``python -m paper_2508_16522_b200.roofline`` prints
JSON).  Library: libtdmicro.so (csrc/microbench.cu).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

from . import _native as N

_mb = None


def _lib():
    global _mb
    if _mb is None:
        if not os.path.exists(N.MB_LIB_PATH):
            raise N.DeviceError(f"{N.MB_LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(N.MB_LIB_PATH)
        L.td_mb_atomic_rate.restype = C.c_double
        L.td_mb_atomic_rate.argtypes = [C.c_int] * 6
        L.td_mb_flag_latency.restype = C.c_double
        L.td_mb_flag_latency.argtypes = [C.c_int, C.c_int, C.c_int]
        L.td_mb_launch_latency.restype = C.c_double
        L.td_mb_launch_latency.argtypes = [C.c_int, C.c_int, C.c_int]
        L.td_mb_p2p_latency.restype = C.c_double
        L.td_mb_p2p_latency.argtypes = [C.c_int, C.c_int, C.c_int]
        L.td_mb_mailbox_hop.restype = C.c_double
        L.td_mb_mailbox_hop.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int]
        L.td_mb_mailbox_hop_strided.restype = C.c_double
        L.td_mb_mailbox_hop_strided.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int]
        L.td_mb_p2p_mailbox_hop.restype = C.c_double
        L.td_mb_p2p_mailbox_hop.argtypes = [C.c_int, C.c_int, C.c_int]
        L.td_mb_dsmem_hop.restype = C.c_double
        L.td_mb_dsmem_hop.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.td_mb_chain_floor.restype = C.c_double
        L.td_mb_chain_floor.argtypes = [C.c_int, C.c_int, C.c_int]
        L.td_mb_compute_peak.restype = C.c_double
        L.td_mb_compute_peak.argtypes = [C.c_int] * 6
        L.td_mb_compute_peak_sustained.restype = C.c_double
        L.td_mb_compute_peak_sustained.argtypes = [C.c_int] * 5 + [C.c_double]
        L.td_mb_last_error.restype = C.c_char_p
        _mb = L
    return _mb


def _chk(x: float) -> float:
    if x < 0:
        raise N.DeviceError(_lib().td_mb_last_error().decode())
    return x


def compute_peak(device: int = 0, sm_count: int = 148, iters: int = 1 << 15, reps: int = 5,
                 sustained_s: float = 3.0) -> dict:
    """Chip peak of the compute_bound body's work unit (u64 LCG lane-updates/s,
    SURVEY Appendix B), the fixed METG denominator (efficiency
    is relative to the machine's peak, not to a configuration's own best).
    Best over 2 / 4 / 8 independent chains per thread at the executor's lean
    geometry (8 x 128-thread CTAs per SM); the 2-chain figure is the executor
    body's own shape (64 lanes per task = 2 per thread)."""
    L = _lib()
    by_chains = {k: _chk(L.td_mb_compute_peak(device, k, 8 * sm_count, 128, iters, reps)) for k in (2, 4, 8)}
    # one warp alone on its SM running the executor body's shape (2 chains per
    # lane): the peak of ONE executor, for configurations with few executors
    per_warp = _chk(L.td_mb_compute_peak(device, 2, sm_count, 32, iters, reps)) / sm_count
    best = max(by_chains, key=lambda k: by_chains[k])
    # sustained: the best chain count back to back for `sustained_s` (clocks
    # settle under the load's power draw, as in a long METG sweep)
    sus = _chk(L.td_mb_compute_peak_sustained(device, best, 8 * sm_count, 128, iters * 4, sustained_s)) \
        if sustained_s > 0 else None
    return {"lane_updates_per_s": by_chains[best], "by_chains": by_chains,
            "sustained_lane_updates_per_s": sus, "sustained_seconds": sustained_s,
            "per_warp_2chain_lane_updates_per_s": per_warp,
            "geometry": "8 CTAs x 128 threads per SM, loop unrolled x8, best of %d (burst)" % reps}


def measure(device: int = 0, sm_count: int = 148, p2p_peer: int | None = None) -> dict:
    L = _lib()
    blocks = sm_count * 8
    out = dict(
        red_distinct_per_s=_chk(L.td_mb_atomic_rate(device, 0, 0, blocks, 256, 64)),
        atom_distinct_per_s=_chk(L.td_mb_atomic_rate(device, 1, 0, blocks, 256, 64)),
        red_same_addr_per_s=_chk(L.td_mb_atomic_rate(device, 0, 1, sm_count, 256, 16)),
        flag_hop_ns=_chk(L.td_mb_flag_latency(device, 20000, 0)),
        hop_red_release_ns=_chk(L.td_mb_flag_latency(device, 20000, 1)),
        hop_token_fence_red_ns=_chk(L.td_mb_flag_latency(device, 20000, 2)),
        hop_token_red_release_ns=_chk(L.td_mb_flag_latency(device, 20000, 3)),
        hop_token_st_release_ns=_chk(L.td_mb_flag_latency(device, 20000, 4)),
        launch_us=_chk(L.td_mb_launch_latency(device, 0, 2000)),
        graph_node_us=_chk(L.td_mb_launch_latency(device, 1, 2000)),
    )
    mn = C.c_double()
    # the message hop over 74 concurrent SM pairs: the minimum is the floor
    # (232-246 ns on every box and word layout measured); the median depends
    # on where the pairs' words and SMs sit (272-480 ns), which is why the
    # 16-pair median used as L_level until round 2 moved 258..434 ns between
    # boxes (scripts/hop_variants.cu)
    med = _chk(L.td_mb_mailbox_hop(device, 74, 20000, C.byref(mn), 0))
    out["mailbox_hop_ns"] = mn.value
    out["mailbox_hop_median_ns"] = med
    out["mailbox_hop_16pairs_median_ns"] = _chk(L.td_mb_mailbox_hop(device, 16, 20000, C.byref(mn), 0))
    out["mailbox_hop_sys_scope_ns"] = _chk(L.td_mb_mailbox_hop(device, 16, 20000, C.byref(mn), 1))
    # the same message as a red.add.u64 into the receiver's shared memory:
    # across the CTAs of a cluster (DSMEM) and between two warps of one CTA
    out["dsmem_hop_ns"] = _chk(L.td_mb_dsmem_hop(device, 16, 20000, 0, C.byref(mn)))
    out["dsmem_hop_min_ns"] = mn.value
    out["cta_smem_hop_ns"] = _chk(L.td_mb_dsmem_hop(device, 16, 20000, 1, C.byref(mn)))
    # floor of a node's own dependent arithmetic (token rule, compute_bound(1)
    # body, ring-fed): cycles per node with 1 and with 7 warps per SM
    out["node_chain_floor_cycles"] = _chk(L.td_mb_chain_floor(device, sm_count, 20000))
    out["node_chain_floor_cycles_7w"] = _chk(L.td_mb_chain_floor(device, 7 * sm_count, 20000))
    if p2p_peer is not None:
        out["p2p_hop_ns"] = _chk(L.td_mb_p2p_latency(device, p2p_peer, 5000))
        out["p2p_mailbox_hop_ns"] = _chk(L.td_mb_p2p_mailbox_hop(device, p2p_peer, 5000))
    return out


if __name__ == "__main__":
    peer = int(sys.argv[1]) if len(sys.argv) > 1 else None
    print(json.dumps(measure(p2p_peer=peer), indent=1))
