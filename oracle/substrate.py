"""Locate the reference's machine substrate — TEST INFRASTRUCTURE.

The CPU reference executor (alg1_cpu.py) runs on the reference's own
``taskdual.machine`` (machine.py:305-465), imported unmodified from, in order:
  1. ``baseline/_ref`` (offline pip install of /root/reference/pkg; git-ignored,
     travels to the GPU box with the snapshot),
  2. ``/root/reference/pkg/src`` (this build container only).
If neither exists, :func:`load` raises; callers report it (no substitute
substrate is used, so a CPU-baseline number always means the real one).
"""
from __future__ import annotations

import importlib
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(_REPO, "baseline", "_ref"), "/root/reference/pkg/src")


def load():
    """Return (machine_module, errors_module, origin_path)."""
    last = None
    for path in CANDIDATES:
        if os.path.isdir(os.path.join(path, "taskdual")):
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                m = importlib.import_module("taskdual.machine")
                e = importlib.import_module("taskdual.errors")
                return m, e, path
            except Exception as exc:  # pragma: no cover
                last = exc
    raise ImportError(f"taskdual.machine not found in {CANDIDATES}: {last}")


def available() -> bool:
    try:
        load()
        return True
    except ImportError:
        return False
