"""numpy restatement of the config-5 mini-app (independent of seq_oracle.c) —
TEST INFRASTRUCTURE.  Same definition as td_oracle_stencil2d."""
import numpy as np

from . import tokens as T


def run(nx: int, ny: int, steps: int, seed: int = 0):
    t = 64
    idx = np.arange(nx * ny, dtype=np.uint64).reshape(ny, nx)
    with np.errstate(over="ignore"):
        a = T.mix64(np.uint64(seed) ^ (idx + np.uint64(T.G2))).astype(np.uint32)
    k = np.arange(t * t, dtype=np.uint64).reshape(t, t)
    w = 2 * k + 1
    rs = []
    for step in range(steps):
        if step > 0:
            p = np.pad(a, 1)
            with np.errstate(over="ignore"):
                a = (np.uint32(2) * a + p[:-2, 1:-1] + p[2:, 1:-1] + p[1:-1, :-2] + p[1:-1, 2:]).astype(np.uint32)
        tiles = a.reshape(ny // t, t, nx // t, t).transpose(0, 2, 1, 3).astype(np.uint64)
        with np.errstate(over="ignore"):
            rs.append((tiles * w).sum(axis=(2, 3), dtype=np.uint64).reshape(-1))
    return np.concatenate(rs), a
