"""Task Bench harness on the GPU executor: ``run_bench`` and ``compute_metg``
(SPEC.md bench 495-562; §6.1 METG definition 961-972).

* A Sample is one granularity point: median device wall time over
  ``repetitions`` replays after ``warmups``.
* granularity = wall * executors / tasks (Task Bench's definition: the mean
  time one executor spends per task; executors = resident worker warps).
* useful-work rate = tasks * iterations * 64 lane-updates / wall for the
  COMPUTE body; efficiency = rate / peak.  The peak is
  either a FIXED reference -- the chip's measured peak for this body
  (``roofline.compute_peak``; PAPER.md:951-965 normalises to the machine's
  peak, so every executor configuration is scored against the same number)
  -- or, when none is given, the best rate of the sweep.
* METG(target) = smallest measured granularity with efficiency >= target,
  no interpolation.
* Every sweep point can be checked: ``run_bench(check=...)`` replays once more
  with column checksums on and compares them with the checker's (the bench
  passes the oracle's); ``Sample.digest_ok`` records the outcome.
"""
from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field

import numpy as np

from .executor import DeviceGraph, device_info
from .flat import KIND_COMPUTE
from .taskbench import generate_graph


@dataclass
class Sample:
    granularity_ns: float   # measured mean time per task per executor
    wall_ns: float          # median wall (device) time of one replay
    rate: float             # useful work per second
    efficiency: float = 0.0
    iterations: int = 0
    tasks: int = 0
    executors: int = 0
    steps: int = 0                  # timesteps of the replayed graph
    digest_ok: bool | None = None   # column checksums == the checker's (None: not checked)


@dataclass
class MetgResult:
    curve: list = field(default_factory=list)   # Samples sorted by granularity
    metg_ns: float | None = None
    peak_rate: float = 0.0
    peak_is_reference: bool = False             # True: a fixed (chip) peak, not the sweep's best


def compute_metg(samples, target: float = 0.5, peak: float | None = None) -> MetgResult:
    """SPEC.md:536-544.  ``samples`` are Sample objects or
    (granularity, efficiency) pairs (efficiency already computed).  ``peak``:
    a fixed reference rate (the chip's measured peak for the body); None =
    the best rate of the samples."""
    samples = list(samples)
    if not samples:
        raise ValueError("compute_metg needs at least one sample")
    ref = peak is not None
    if not isinstance(samples[0], Sample):
        curve = [Sample(granularity_ns=float(g), wall_ns=0.0, rate=float(e), efficiency=float(e))
                 for g, e in samples]
        peak = max(s.rate for s in curve) if peak is None else float(peak)
        if ref:
            curve = [Sample(**{**s.__dict__, "efficiency": s.rate / peak}) for s in curve]
    else:
        peak = max(s.rate for s in samples) if peak is None else float(peak)
        curve = [Sample(**{**s.__dict__, "efficiency": (s.rate / peak if peak > 0 else 0.0)})
                 for s in samples]
    curve.sort(key=lambda s: s.granularity_ns)
    metg = None
    for s in curve:
        if s.efficiency >= target:
            metg = s.granularity_ns
            break
    return MetgResult(curve=curve, metg_ns=metg, peak_rate=peak, peak_is_reference=ref)


@dataclass
class BenchConfig:
    """SPEC.md:504-507, GPU form."""
    pattern: str = "stencil_1d"
    width: int = 1024
    steps: int = 1000
    iterations: tuple = tuple(1 << k for k in range(0, 21))
    repetitions: int = 5
    warmups: int = 2
    n_workers: int | None = None
    mapping: str = "block"
    device: int = 0
    seed: int = 0
    # one replay is kept under this wall time: beyond it the graph is replayed
    # with fewer timesteps (recorded per sample as Sample.steps)
    max_replay_ms: float = 60.0
    radix: int = 5
    # stop once the efficiency has saturated: the last `plateau` points'
    # rates within `plateau_tol` of each other (0 = sweep every point)
    plateau: int = 0
    plateau_tol: float = 0.02


def _steps_for(cfg: BenchConfig, iters: int, base_step_us: float, us_per_iter: float) -> int:
    est = base_step_us + us_per_iter * iters
    cap = int(cfg.max_replay_ms * 1e3 / max(est, 1e-3))
    return int(max(min(cfg.steps, cap), 8))


def run_bench(cfg: BenchConfig, verbose: bool = False, check=None) -> list[Sample]:
    """Sweep the COMPUTE body over cfg.iterations.

    The graph is uploaded once per length class and re-parameterised in place
    (``set_body_arg``) for each granularity; the number of timesteps stays at
    cfg.steps unless one replay would exceed ``max_replay_ms``.

    ``check(graph, iterations) -> expected column checksums`` (or None to skip
    the point): after the timed replays, one more replay with checksums on is
    compared with it (``Sample.digest_ok``)."""
    info = device_info(cfg.device)
    workers = min(cfg.n_workers or cfg.width, info["max_workers"], cfg.width)
    samples = []
    base_step_us, us_per_iter = 1.5, 0.006
    graphs: dict[int, tuple] = {}
    try:
        for it in cfg.iterations:
            cap = _steps_for(cfg, it, base_step_us, us_per_iter)
            classes = sorted({cfg.steps, min(cfg.steps, 256), min(cfg.steps, 64), min(cfg.steps, 16)},
                             reverse=True)
            steps = next((c for c in classes if c <= cap), classes[-1])  # few distinct lengths
            if steps not in graphs:
                g = generate_graph(cfg.pattern, cfg.width, steps, radix=cfg.radix, n_workers=workers,
                                   mapping=cfg.mapping, kind=KIND_COMPUTE, arg=1)
                graphs[steps] = (g, DeviceGraph(g, cfg.device))
            g, dg = graphs[steps]
            dg.set_body_arg(it)
            for _ in range(cfg.warmups):
                dg.run(cfg.seed, flags=0)
            ts = []
            for _ in range(cfg.repetitions):
                dg.run(cfg.seed, flags=0)
                ts.append(dg.last_ms())
            wall_ms = float(np.median(ts))
            wall_ns = wall_ms * 1e6
            rate = g.n * it * 64 / (wall_ms * 1e-3)
            gran = wall_ns * workers / g.n
            ok = None
            want = check(g, it) if check is not None else None
            if want is not None:
                from . import _native as N
                dg.run(cfg.seed, flags=N.TD_F_CHECKSUM)
                ok = bool(np.array_equal(dg.checksums(), want))
            samples.append(Sample(granularity_ns=gran, wall_ns=wall_ns, rate=rate, iterations=it,
                                  tasks=g.n, executors=workers, steps=steps, digest_ok=ok))
            if it <= 2:
                base_step_us = wall_ms * 1e3 / steps
            else:
                us_per_iter = max((wall_ms * 1e3 / steps - base_step_us) / it, 1e-5)
            if verbose:
                print(f"  iters={it:>8} steps={steps:>5} wall={wall_ms:9.3f} ms gran={gran/1e3:9.3f} us "
                      f"rate={rate:.3e} digest={ok}", flush=True)
            if cfg.plateau and len(samples) >= cfg.plateau:
                last = [x.rate for x in samples[-cfg.plateau:]]
                if max(last) <= (1 + cfg.plateau_tol) * min(last):
                    break
    finally:
        for _, dg in graphs.values():
            dg.close()
    return samples


def to_csv(system: str, cfg: BenchConfig, result: MetgResult) -> str:
    """CSV schema of SPEC.md:557 (+ iterations, executors)."""
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(["system", "pattern", "width", "steps", "granularity_ns", "wall_ns", "rate", "efficiency",
                "iterations", "executors", "digest_ok"])
    for s in result.curve:
        w.writerow([system, cfg.pattern, cfg.width, s.steps or s.tasks // max(cfg.width, 1),
                    f"{s.granularity_ns:.1f}", f"{s.wall_ns:.1f}", f"{s.rate:.6e}", f"{s.efficiency:.4f}",
                    s.iterations, s.executors, "" if s.digest_ok is None else int(s.digest_ok)])
    return buf.getvalue()
