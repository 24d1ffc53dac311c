"""Task Bench harness on the GPU executor: ``run_bench`` and ``compute_metg``
(SPEC.md bench 495-562; §6.1 METG definition 961-972).

* A Sample is one granularity point: median device wall time over
  ``repetitions`` replays after ``warmups``.
* granularity = wall * executors / tasks (Task Bench's definition: the mean
  time one executor spends per task; executors = resident worker warps).
* useful-work rate = tasks * iterations * 64 lane-updates / wall for the
  COMPUTE body; efficiency = rate / peak, peak = best
  rate measured in the sweep.
* METG(target) = smallest measured granularity with efficiency >= target,
  no interpolation.
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


@dataclass
class MetgResult:
    curve: list = field(default_factory=list)   # Samples sorted by granularity
    metg_ns: float | None = None
    peak_rate: float = 0.0


def compute_metg(samples, target: float = 0.5) -> MetgResult:
    """SPEC.md:536-544.  ``samples`` are Sample objects or
    (granularity, efficiency) pairs (efficiency already computed)."""
    samples = list(samples)
    if not samples:
        raise ValueError("compute_metg needs at least one sample")
    if not isinstance(samples[0], Sample):
        curve = [Sample(granularity_ns=float(g), wall_ns=0.0, rate=float(e), efficiency=float(e))
                 for g, e in samples]
        peak = max(s.rate for s in curve)
    else:
        peak = max(s.rate for s in samples)
        curve = [Sample(**{**s.__dict__, "efficiency": (s.rate / peak if peak > 0 else 0.0)})
                 for s in samples]
    curve.sort(key=lambda s: s.granularity_ns)
    metg = None
    for s in curve:
        if s.efficiency >= target:
            metg = s.granularity_ns
            break
    return MetgResult(curve=curve, metg_ns=metg, peak_rate=peak)


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
    max_replay_ms: float = 60.0     # cap steps at large iteration counts
    radix: int = 5


def _steps_for(cfg: BenchConfig, iters: int, base_step_us: float, us_per_iter: float) -> int:
    est = base_step_us + us_per_iter * iters
    cap = int(cfg.max_replay_ms * 1e3 / max(est, 1e-3))
    return int(max(min(cfg.steps, cap), 8))


def run_bench(cfg: BenchConfig, verbose: bool = False) -> list[Sample]:
    """Sweep the COMPUTE body over cfg.iterations.

    The graph is uploaded once per length class and re-parameterised in place
    (``set_body_arg``) for each granularity; the number of timesteps shrinks
    for very long bodies so one replay stays near ``max_replay_ms``."""
    info = device_info(cfg.device)
    workers = min(cfg.n_workers or cfg.width, info["max_workers"], cfg.width)
    samples = []
    base_step_us, us_per_iter = 1.5, 0.006
    graphs: dict[int, tuple] = {}
    try:
        for it in cfg.iterations:
            cap = _steps_for(cfg, it, base_step_us, us_per_iter)
            classes = sorted({cfg.steps, min(cfg.steps, 128), min(cfg.steps, 16)}, reverse=True)
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
            samples.append(Sample(granularity_ns=gran, wall_ns=wall_ns, rate=rate, iterations=it,
                                  tasks=g.n, executors=workers))
            if it <= 2:
                base_step_us = wall_ms * 1e3 / steps
            else:
                us_per_iter = max((wall_ms * 1e3 / steps - base_step_us) / it, 1e-5)
            if verbose:
                print(f"  iters={it:>8} steps={steps:>5} wall={wall_ms:9.3f} ms gran={gran/1e3:9.3f} us "
                      f"rate={rate:.3e}", flush=True)
    finally:
        for _, dg in graphs.values():
            dg.close()
    return samples


def to_csv(system: str, cfg: BenchConfig, result: MetgResult) -> str:
    """CSV schema of SPEC.md:557 (+ iterations, executors)."""
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(["system", "pattern", "width", "steps", "granularity_ns", "wall_ns", "rate", "efficiency",
                "iterations", "executors"])
    for s in result.curve:
        w.writerow([system, cfg.pattern, cfg.width, s.tasks // max(cfg.width, 1), f"{s.granularity_ns:.1f}",
                    f"{s.wall_ns:.1f}", f"{s.rate:.6e}", f"{s.efficiency:.4f}", s.iterations, s.executors])
    return buf.getvalue()
