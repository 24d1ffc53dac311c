"""Token, fold and task-body definitions (oracle side) — TEST INFRASTRUCTURE.

The reference leaves the per-task output token and its fold unspecified
("a correctness checksum (per-task output token folded per column)",
SPEC.md:530-531; cross-system equality).
recommends a splitmix64-based token; we fix the following definition, which
is scheduling- and sharding-independent (inputs are identified by node id,
never by arrival order) and whose fold is an exact integer sum, so that each
dependence message can CARRY its input: a producer u sends every successor
one 64-bit atomic add ``(1 << 48) + term(u)`` into the successor's mailbox
word, whose top 16 bits count arrivals and low 48 bits accumulate the terms.

    h0      = mix64(seed ^ mix64(v + G1))                   v = global node id
    term(u) = mix64(tok[u] ^ mix64(u + G3)) >> 32           32-bit input term
    acc     = sum_{u in preds(v)} term(u)                   exact, < 2^48 (indeg < 2^16)
    h       = mix64(h0 ^ acc)
    r       = body(kind, arg, h)
    tok[v]  = h ^ r

Bodies (arg is a u32 per node):
    EMPTY          r = 0
    BUSY_WAIT(ns)  r = 0           (spins `ns` on the device timer / host clock)
    COMPUTE(iters) r = XOR_{l<64} LCG^iters(mix64(h ^ (l+1)*G2))
                   LCG(x) = A*x + C mod 2^64 (Knuth MMIX constants); useful work
                   is iters*64 lane-updates.
    STENCIL2D      r = fold of the tile's output cells (config 5; see
                   stencil2d.py)
    MEMORY(n)      r = XOR_{k<n} (h + k*G2)   (memory_bound: the device streams
                   these n words through HBM -- stores them, loads them back)

Column checksum = XOR of every token of the column (all timesteps); graph
checksum = XOR over columns.  Parity is judged on the full token array.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
G1 = 0x9E3779B97F4A7C15
G2 = 0xD1B54A32D192ED03
G3 = 0x8CB92BA72F3D8DD7
MAX_INDEG = (1 << 16) - 1
LCG_A = 6364136223846793005
LCG_C = 1442695040888963407

BODY_EMPTY = 0
BODY_BUSY_WAIT = 1
BODY_COMPUTE = 2
BODY_STENCIL2D = 3
BODY_MEMORY = 6
N_LANES = 64

_U = np.uint64


def mix64_int(z: int) -> int:
    """splitmix64 finaliser on a Python int (mod 2^64)."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix64(z: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on a uint64 array (wraps mod 2^64)."""
    z = np.asarray(z, dtype=_U)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U(30))) * _U(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
    return z ^ (z >> _U(31))


def affine_pow(n: int) -> tuple[int, int]:
    """(A_n, C_n) with LCG^n(x) = A_n*x + C_n mod 2^64.

    Binary exponentiation of map composition (A,C)o(A',C') = (A*A', A*C'+C);
    the closed form c*(a^n-1)/(a-1) is NOT usable mod 2^64 (a-1 is even).
    """
    ra, rc = 1, 0          # identity
    ba, bc = LCG_A, LCG_C  # LCG^1
    while n:
        if n & 1:
            # r <- b o r
            ra, rc = (ba * ra) & M64, (ba * rc + bc) & M64
        # b <- b o b
        ba, bc = (ba * ba) & M64, (ba * bc + bc) & M64
        n >>= 1
    return ra, rc


def lcg_iter_int(x: int, n: int) -> int:
    """The literal loop (used by small tests to check affine_pow)."""
    for _ in range(n):
        x = (LCG_A * x + LCG_C) & M64
    return x


with np.errstate(over="ignore"):
    _LANE_KEYS = np.arange(1, N_LANES + 1, dtype=_U) * _U(G2)


def compute_body(h: np.ndarray, iters: np.ndarray) -> np.ndarray:
    """COMPUTE(iters) body result for arrays of h (uint64) and iters (int)."""
    h = np.asarray(h, dtype=_U)
    iters = np.broadcast_to(np.asarray(iters, dtype=np.int64), h.shape)
    out = np.zeros(h.shape, dtype=_U)
    if h.size == 0:
        return out
    with np.errstate(over="ignore"):
        x0 = mix64(h[..., None] ^ _LANE_KEYS)  # (..., 64)
        for n in np.unique(iters):
            a, c = affine_pow(int(n))
            sel = iters == n
            xn = x0[sel] * _U(a) + _U(c)
            out[sel] = np.bitwise_xor.reduce(xn, axis=-1)
    return out


def compute_body_int(h: int, iters: int) -> int:
    a, c = affine_pow(iters)
    r = 0
    for lane in range(N_LANES):
        x = mix64_int(h ^ (((lane + 1) * G2) & M64))
        r ^= (a * x + c) & M64
    return r


def memory_body(h: np.ndarray, words: np.ndarray) -> np.ndarray:
    """MEMORY(n) body result r = XOR_{k<n} (h + k*G2) (uint64 arrays)."""
    h = np.asarray(h, dtype=_U)
    words = np.broadcast_to(np.asarray(words, dtype=np.int64), h.shape)
    out = np.zeros(h.shape, dtype=_U)
    with np.errstate(over="ignore"):
        for i in np.ndindex(h.shape):
            k = np.arange(int(words[i]), dtype=_U)
            out[i] = np.bitwise_xor.reduce(h[i] + k * _U(G2)) if k.size else _U(0)
    return out


def memory_body_int(h: int, words: int) -> int:
    r = 0
    for k in range(words):
        r ^= (h + k * G2) & M64
    return r


def task_h0(seed: int, ids: np.ndarray) -> np.ndarray:
    ids = np.asarray(ids, dtype=_U)
    with np.errstate(over="ignore"):
        return mix64(_U(seed & M64) ^ mix64(ids + _U(G1)))


def input_term(tokens: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """term(u) = mix64(tok[u] ^ mix64(u + G3)) >> 32 (uint64 arrays)."""
    with np.errstate(over="ignore"):
        k = mix64(np.asarray(ids, dtype=_U) + _U(G3))
    return mix64(np.asarray(tokens, dtype=_U) ^ k) >> _U(32)


def term_int(tok: int, u: int) -> int:
    return mix64_int((tok & M64) ^ mix64_int(u + G3)) >> 32


def finish_token(h0: np.ndarray, acc: np.ndarray, kind: np.ndarray, arg: np.ndarray,
                 body_extra: np.ndarray | None = None) -> np.ndarray:
    """tok = h ^ body(h) with h = mix64(h0 ^ acc)."""
    h = mix64(np.asarray(h0, dtype=_U) ^ np.asarray(acc, dtype=_U))
    kind = np.broadcast_to(np.asarray(kind), h.shape)
    arg = np.broadcast_to(np.asarray(arg), h.shape)
    r = np.zeros(h.shape, dtype=_U)
    sel = kind == BODY_COMPUTE
    if sel.any():
        r[sel] = compute_body(h[sel], arg[sel])
    sel = kind == BODY_MEMORY
    if sel.any():
        r[sel] = memory_body(h[sel], arg[sel])
    if body_extra is not None:
        r ^= np.asarray(body_extra, dtype=_U)
    return h ^ r


def token_int(seed: int, v: int, pred_tokens: dict | list, kind: int = BODY_EMPTY,
              arg: int = 0) -> int:
    """Scalar restatement (pure Python) used by the small-graph oracle.
    ``pred_tokens`` maps predecessor id -> token (or is a list of (id, token))."""
    items = pred_tokens.items() if isinstance(pred_tokens, dict) else pred_tokens
    h0 = mix64_int((seed & M64) ^ mix64_int(v + G1))
    acc = 0
    for u, t in items:
        acc += term_int(t, u)
    h = mix64_int(h0 ^ acc)
    r = compute_body_int(h, arg) if kind == BODY_COMPUTE else memory_body_int(h, arg) if kind == BODY_MEMORY else 0
    return h ^ r


def column_checksums(tokens: np.ndarray, width: int) -> np.ndarray:
    """XOR of every token per column for a (steps*width) Task Bench array."""
    t = np.asarray(tokens, dtype=_U).reshape(-1, width)
    return np.bitwise_xor.reduce(t, axis=0)
