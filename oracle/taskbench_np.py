"""numpy per-timestep Task Bench oracle — TEST INFRASTRUCTURE.

An independent restatement (it does not import the product's generator) of
  * the Task Bench dependence patterns: SPEC.md:500-503 (stencil radius 1,
    independent) and SURVEY.md Appendix A for the extended patterns (not in
    the reference; parity unpinned by it),
  * node ids t*width + c (dense cumulative offsets for tree),
  * the token fold of oracle/tokens.py (builder definition).

Because every edge goes from step t-1 to step t, a node's token depends only
on the previous step's tokens, so the sequential topological oracle of
SPEC.md:224/408 collapses to one vectorised pass per timestep.
"""
from __future__ import annotations

import math

import numpy as np

from . import tokens as T


def _L(W: int) -> int:
    return max(1, math.ceil(math.log2(W))) if W > 1 else 1


def width_at(pattern: str, W: int, t: int) -> int:
    return min(W, 1 << min(t, 62)) if pattern == "tree" else W


def deps(pattern: str, W: int, t: int, p: int, radix: int = 5) -> list[int]:
    """Dependence points of (t, p) in step t-1, ascending (scalar restatement)."""
    if t == 0:
        return []
    pat = {"independent": "trivial", "stencil": "stencil_1d"}.get(pattern, pattern)
    wprev = width_at(pat, W, t - 1)
    if pat == "trivial":
        return []
    if pat == "no_comm":
        return [p] if p < wprev else []
    if pat == "stencil_1d":
        return [q for q in (p - 1, p, p + 1) if 0 <= q < W]
    if pat == "stencil_1d_periodic":
        return sorted({(p - 1) % W, p, (p + 1) % W})
    if pat == "tree":
        return [p // 2] if p // 2 < wprev else []
    if pat == "nearest":
        return list(range(max(0, p - (radix - 1) // 2), min(W - 1, p + radix // 2) + 1))
    if pat == "fft":
        s = 1 << ((t + _L(W) - 1) % _L(W))
        return [q for q in (p - s, p, p + s) if 0 <= q < W]
    if pat == "spread":
        ds = (t + _L(W) - 1) % _L(W)
        return sorted({(p + i * (W // radix) + (ds if i > 0 else 0)) % W for i in range(radix)})
    if pat == "all_to_all":
        return list(range(W))
    raise ValueError(pattern)


def run(pattern: str, W: int, steps: int, seed: int = 0, kind: int = T.BODY_EMPTY,
        arg: int = 0, radix: int = 5) -> np.ndarray:
    """Full token array (node-id order) for a Task Bench graph."""
    pat = {"independent": "trivial", "stencil": "stencil_1d"}.get(pattern, pattern)
    out = []
    prev = None
    off = 0
    for t in range(steps):
        w = width_at(pat, W, t)
        ids = np.arange(off, off + w, dtype=np.uint64)
        h0 = T.task_h0(seed, ids)
        acc = np.zeros(w, dtype=np.uint64)
        if t > 0 and pat != "trivial":
            prev_ids = np.arange(off - len(prev), off, dtype=np.uint64)
            terms_prev = T.input_term(prev, prev_ids)      # term(u) for every u of step t-1
            if pat == "all_to_all":
                acc[:] = terms_prev.sum(dtype=np.uint64)   # every point folds all of step t-1
            else:
                rows = [deps(pat, W, t, p, radix) for p in range(w)]
                k = max((len(r) for r in rows), default=0)
                if k:
                    mat = np.full((w, k), -1, dtype=np.int64)
                    for p, r in enumerate(rows):
                        mat[p, : len(r)] = r
                    valid = mat >= 0
                    terms = terms_prev[np.where(valid, mat, 0)]
                    terms[~valid] = 0
                    acc = terms.sum(axis=1, dtype=np.uint64)
        cur = T.finish_token(h0, acc, kind, arg)
        out.append(cur)
        prev = cur
        off += w
    return np.concatenate(out)


def column_checksums(pattern: str, W: int, steps: int, tokens: np.ndarray) -> np.ndarray:
    cols = np.concatenate([np.arange(width_at(pattern, W, t)) for t in range(steps)])
    out = np.zeros(W, dtype=np.uint64)
    np.bitwise_xor.at(out, cols, tokens)
    return out
