"""Task Bench graph generators emitting the flat interval CSR directly.

Reference: bench ``generate_graph(pattern, mapping)``: node
ids ``t*width + c``, stencil(radius=1) and independent
(SPEC.md:500-503), column->processor mapping round-robin by default
(SPEC.md:505).  The extended patterns named by BASELINE.json's configs
(no_comm, fft, tree, nearest, all_to_all, spread) are NOT in the reference;
they follow the public Task Bench definitions restated in SURVEY.md
Appendix A (parity unpinned by the reference; pinned by our golden vectors).

Every dependence set is produced as sorted, disjoint id intervals, and the
successor side is produced analytically (Task Bench's reverse dependencies),
so all_to_all at W=8192 costs one interval per node rather than W ids.
"""
from __future__ import annotations

import math

import numpy as np

from .flat import FlatGraph, IntervalCSR, KIND_EMPTY, transpose

PATTERNS = (
    "trivial", "independent", "no_comm", "stencil_1d", "stencil", "stencil_1d_periodic",
    "tree", "fft", "nearest", "spread", "all_to_all",
)


def _canon(pattern: str) -> str:
    p = pattern.lower()
    if p == "independent":  # SPEC.md:501 'independent' == Task Bench 'trivial'
        return "trivial"
    if p == "stencil":      # SPEC.md:502 stencil(radius=1)
        return "stencil_1d"
    if p not in PATTERNS:
        raise ValueError(f"unknown pattern {pattern!r}")
    return p


def n_dependence_sets(width: int) -> int:
    return max(1, math.ceil(math.log2(width))) if width > 1 else 1


def dset_at(t: int, width: int) -> int:
    L = n_dependence_sets(width)
    return (t + L - 1) % L


def width_at(pattern: str, width: int, t: int) -> int:
    if _canon(pattern) == "tree":
        return min(width, 1 << min(t, 62))
    return width


def offsets(pattern: str, width: int, steps: int) -> np.ndarray:
    w = np.array([width_at(pattern, width, t) for t in range(steps)], dtype=np.int64)
    off = np.zeros(steps + 1, dtype=np.int64)
    np.cumsum(w, out=off[1:])
    return off


def _deps_points(pattern: str, width: int, t: int, p: np.ndarray, radix: int):
    """Candidate dependence intervals in POINT space of step t-1.
    Returns (lo[n,k], hi[n,k], valid[n,k]) sorted per row."""
    pat = _canon(pattern)
    W = width
    wprev = width_at(pat, W, t - 1)
    one = lambda lo, hi, ok: (lo[:, None], hi[:, None], ok[:, None])  # noqa: E731
    if pat == "trivial":
        z = np.zeros((len(p), 0), dtype=np.int64)
        return z, z, z.astype(bool)
    if pat == "no_comm":
        return one(p, p, p < wprev)
    if pat == "stencil_1d":
        return one(np.maximum(p - 1, 0), np.minimum(p + 1, W - 1), np.ones(len(p), bool))
    if pat == "stencil_1d_periodic":
        if W <= 3:
            lo = np.zeros((len(p), 1), np.int64)
            return lo, lo + (W - 1), np.ones((len(p), 1), bool)
        c = np.sort(np.stack([(p - 1) % W, p, (p + 1) % W], axis=1), axis=1)
        return c, c, np.ones(c.shape, bool)
    if pat == "tree":
        q = p // 2
        return one(q, q, q < wprev)
    if pat == "nearest":
        return one(np.maximum(p - (radix - 1) // 2, 0), np.minimum(p + radix // 2, W - 1),
                   np.ones(len(p), bool))
    if pat == "fft":
        s = 1 << dset_at(t, W)
        c = np.stack([p - s, p, p + s], axis=1)
        ok = (c >= 0) & (c < W)
        return c, c, ok
    if pat == "all_to_all":
        return one(np.zeros_like(p), np.full_like(p, W - 1), np.ones(len(p), bool))
    if pat == "spread":
        ds = dset_at(t, W)
        i = np.arange(radix)
        c = (p[:, None] + i[None, :] * (W // radix) + np.where(i > 0, ds, 0)[None, :]) % W
        c = np.sort(c, axis=1)
        ok = np.ones(c.shape, bool)
        ok[:, 1:] = c[:, 1:] != c[:, :-1]  # drop duplicates
        return c, c, ok
    raise ValueError(pattern)


def _rdeps_points(pattern: str, width: int, t: int, p: np.ndarray, radix: int):
    """Candidate successor intervals in POINT space of step t+1 (Task Bench
    reverse dependencies)."""
    pat = _canon(pattern)
    W = width
    wnext = width_at(pat, W, t + 1)
    one = lambda lo, hi, ok: (lo[:, None], hi[:, None], ok[:, None])  # noqa: E731
    if pat == "trivial":
        z = np.zeros((len(p), 0), dtype=np.int64)
        return z, z, z.astype(bool)
    if pat == "no_comm":
        return one(p, p, p < wnext)
    if pat in ("stencil_1d", "stencil_1d_periodic", "fft"):
        return _deps_points(pat, W, t + 1, p, radix)  # symmetric sets
    if pat == "tree":
        return one(2 * p, np.minimum(2 * p + 1, wnext - 1), 2 * p < wnext)
    if pat == "nearest":
        return one(np.maximum(p - radix // 2, 0), np.minimum(p + (radix - 1) // 2, W - 1),
                   np.ones(len(p), bool))
    if pat == "all_to_all":
        return one(np.zeros_like(p), np.full_like(p, W - 1), np.ones(len(p), bool))
    raise NotImplementedError(pat)


def _pack(n: int, lo: np.ndarray, hi: np.ndarray, ok: np.ndarray) -> IntervalCSR:
    """Rows of sorted candidate id intervals -> merged interval CSR."""
    k = lo.shape[1] if lo.ndim == 2 else 0
    if k == 0:
        return IntervalCSR(np.zeros(n + 1, np.int64), np.zeros((0, 2), np.int32))
    node = np.repeat(np.arange(n, dtype=np.int64)[:, None], k, axis=1)[ok]
    lo, hi = lo[ok], hi[ok]
    if len(node) == 0:  # no edges at all (e.g. steps == 1: every task is a source)
        return IntervalCSR(np.zeros(n + 1, np.int64), np.zeros((0, 2), np.int32))
    start = np.ones(len(node), dtype=bool)
    if len(node) > 1:
        start[1:] = (node[1:] != node[:-1]) | (lo[1:] != hi[:-1] + 1)
    sidx = np.flatnonzero(start)
    eidx = np.append(sidx[1:], len(node)) - 1
    iv = np.stack([lo[sidx], hi[eidx]], axis=1).astype(np.int32)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(node[sidx], minlength=n), out=ptr[1:])
    return IntervalCSR(ptr, iv)


def generate_graph(pattern: str, width: int, steps: int, *, radix: int = 5,
                   n_workers: int | None = None, mapping: str = "block",
                   kind: int = KIND_EMPTY, arg: int = 0) -> FlatGraph:
    """Task Bench graph as a FlatGraph.

    mapping: 'round_robin' (SPEC.md:505 default: column c -> worker c % P) or
    'block' (column c -> worker c*P//W; keeps neighbouring columns on one SM).
    """
    if width < 1 or steps < 1:
        raise ValueError("width and steps must be >= 1")
    pat = _canon(pattern)
    off = offsets(pat, width, steps)
    n = int(off[-1])
    P = width if n_workers is None else int(n_workers)
    if P < 1:
        raise ValueError("n_workers must be >= 1")
    t_of = np.repeat(np.arange(steps, dtype=np.int64), np.diff(off))
    p_of = np.arange(n, dtype=np.int64) - off[t_of]

    # dependence candidates per step (the candidate count k is step-invariant)
    plo, phi, pok, slo, shi, sok = [], [], [], [], [], []
    analytic_succ = pat != "spread"
    for t in range(steps):
        p = np.arange(width_at(pat, width, t), dtype=np.int64)
        if t == 0:
            lo, hi, ok = _deps_points(pat, width, 1, p, radix)
            lo, hi, ok = lo[:, :0], hi[:, :0], ok[:, :0]
            k = _deps_points(pat, width, 1, np.zeros(1, np.int64), radix)[0].shape[1]
            lo = np.zeros((len(p), k), np.int64)
            hi = lo.copy()
            ok = np.zeros((len(p), k), bool)
        else:
            lo, hi, ok = _deps_points(pat, width, t, p, radix)
            lo, hi = lo + off[t - 1], hi + off[t - 1]
        plo.append(lo), phi.append(hi), pok.append(ok)
        if analytic_succ:
            if t == steps - 1:
                k = _rdeps_points(pat, width, 0, np.zeros(1, np.int64), radix)[0].shape[1]
                s_lo = np.zeros((len(p), k), np.int64)
                s_hi, s_ok = s_lo.copy(), np.zeros((len(p), k), bool)
            else:
                s_lo, s_hi, s_ok = _rdeps_points(pat, width, t, p, radix)
                s_lo, s_hi = s_lo + off[t + 1], s_hi + off[t + 1]
            slo.append(s_lo), shi.append(s_hi), sok.append(s_ok)
    pred = _pack(n, np.concatenate(plo), np.concatenate(phi), np.concatenate(pok))
    succ = (_pack(n, np.concatenate(slo), np.concatenate(shi), np.concatenate(sok))
            if analytic_succ else transpose(pred))

    if mapping == "round_robin":
        worker = (p_of % P).astype(np.int32)
    elif mapping == "block":
        worker = (p_of * P // width).astype(np.int32)
    else:
        raise ValueError(f"unknown mapping {mapping!r}")
    g = FlatGraph(
        n=n, pred=pred, succ=succ,
        kind=np.full(n, kind, dtype=np.uint8), arg=np.full(n, arg, dtype=np.uint32),
        worker=worker, n_workers=P,
        col=p_of.astype(np.int32), n_cols=width,
        order=np.arange(n, dtype=np.int64),  # ids are a topological order
        meta=dict(pattern=pat, width=width, steps=steps, radix=radix, offsets=off,
                  mapping=mapping),
    )
    return g


def generate_stencil2d(nx: int, ny: int, steps: int, *, tile: int = 64, n_workers: int | None = None,
                       mapping: str = "shard_block", shards: int = 1) -> FlatGraph:
    """BASELINE configs[4] mini-app: a (nx x ny) u32 grid updated by a 5-point
    stencil in (tile x tile) tasks per step (PRK-style).
    Node id t*ntiles + ty*tiles_x + tx; task (t, ty, tx) depends on (t-1, ty, tx)
    and its four neighbours; body TD_BODY_STENCIL2D (step 0 initialises).

    ``mapping``: "block" gives each worker a run of consecutive tiles, "cyclic"
    deals tiles round-robin, and "shard_cyclic" first splits the tiles into
    ``shards`` contiguous row blocks (one per GPU under ShardingPlan.blocks)
    and deals each block round-robin over that shard's workers -- so the tiles
    on a shard boundary, whose halo comes over NVLink, land on distinct
    workers instead of queueing behind each other on a few.  "shard_block"
    keeps the block mapping inside each shard (spatially clustered tiles per
    worker, which the single-GPU run prefers) but spreads the boundary tiles
    evenly through the block order."""
    from .flat import KIND_STENCIL2D
    if nx % tile or ny % tile:
        raise ValueError("grid must be a multiple of the tile size")
    tx_n, ty_n = nx // tile, ny // tile
    nt = tx_n * ty_n
    n = nt * steps
    tiles = np.arange(nt, dtype=np.int64)
    ty, tx = tiles // tx_n, tiles % tx_n
    # candidate predecessor intervals in tile space (sorted): up, [left..right], down
    lo = np.stack([tiles - tx_n, tiles - (tx > 0), tiles + tx_n], axis=1)
    hi = np.stack([tiles - tx_n, tiles + (tx < tx_n - 1), tiles + tx_n], axis=1)
    ok = np.stack([ty > 0, np.ones(nt, bool), ty < ty_n - 1], axis=1)
    plo, phi, pok = [], [], []
    for t in range(steps):
        if t == 0:
            plo.append(np.zeros((nt, 3), np.int64)), phi.append(np.zeros((nt, 3), np.int64))
            pok.append(np.zeros((nt, 3), bool))
        else:
            plo.append(lo + (t - 1) * nt), phi.append(hi + (t - 1) * nt), pok.append(ok)
    pred = _pack(n, np.concatenate(plo), np.concatenate(phi), np.concatenate(pok))
    slo, shi, sok = [], [], []
    for t in range(steps):
        if t == steps - 1:
            slo.append(np.zeros((nt, 3), np.int64)), shi.append(np.zeros((nt, 3), np.int64))
            sok.append(np.zeros((nt, 3), bool))
        else:
            slo.append(lo + (t + 1) * nt), shi.append(hi + (t + 1) * nt), sok.append(ok)
    succ = _pack(n, np.concatenate(slo), np.concatenate(shi), np.concatenate(sok))
    P = nt if n_workers is None else int(n_workers)
    tile_of = np.tile(tiles, steps)
    if mapping == "block":
        worker = tile_of * P // nt
    elif mapping == "cyclic":
        worker = tile_of % P
    elif mapping == "shard_cyclic":
        if P % shards:
            raise ValueError("shard_cyclic needs n_workers divisible by shards")
        pr = P // shards
        r = tile_of * shards // nt
        first = (r * nt + shards - 1) // shards  # first tile of shard r
        worker = r * pr + (tile_of - first) % pr
    elif mapping == "shard_block":
        # per shard: block mapping, with the shard-boundary tiles spread evenly
        # through the block order so each worker gets at most a few of them
        if P % shards:
            raise ValueError("shard_block needs n_workers divisible by shards")
        pr = P // shards
        r_t = tiles * shards // nt
        bnd = np.zeros(nt, bool)
        bnd[ty > 0] |= r_t[tiles[ty > 0] - tx_n] != r_t[ty > 0]
        bnd[ty < ty_n - 1] |= r_t[tiles[ty < ty_n - 1] + tx_n] != r_t[ty < ty_n - 1]
        w_t = np.empty(nt, np.int64)
        for r in range(shards):
            mine = np.flatnonzero(r_t == r)
            S = len(mine)
            b, i = mine[bnd[mine]], mine[~bnd[mine]]
            key = np.empty(S)
            key[:len(b)] = (np.arange(len(b)) + 0.5) * S / max(len(b), 1)
            key[len(b):] = (np.arange(len(i)) + 0.5) * S / max(len(i), 1)
            pos = np.empty(S, np.int64)
            pos[np.argsort(key, kind="stable")] = np.arange(S)
            w_t[np.concatenate([b, i])] = r * pr + pos * pr // S
        worker = w_t[tile_of]
    else:
        raise ValueError(f"unknown mapping {mapping!r}")
    worker = worker.astype(np.int32)
    return FlatGraph(n=n, pred=pred, succ=succ, kind=np.full(n, KIND_STENCIL2D, np.uint8),
                     arg=np.zeros(n, np.uint32), worker=worker, n_workers=P,
                     col=tile_of.astype(np.int32), n_cols=nt, order=np.arange(n, dtype=np.int64),
                     meta=dict(pattern="stencil2d", nx=nx, ny=ny, tile=tile, steps=steps, width=nt))
