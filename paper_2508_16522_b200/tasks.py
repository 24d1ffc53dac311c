"""Task registration (SPEC.md task_rt ``register_task`` 171-179; Fig. 4).

On the CPU a task body is a Python callable.  On the GPU a
body must be a device-body descriptor from the fixed device table
(include/tdexec.h ``TD_BODY_*``): this is the one semantic narrowing of the
API.  Registering a Python callable is allowed (so programs
written for the reference still register), but compiling a graph that uses
it raises :class:`CompileError`.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import CompileError, RegistrationError
from .flat import KIND_BUSY_WAIT, KIND_COMPUTE, KIND_EMPTY, KIND_MEMORY


@dataclass(frozen=True)
class DeviceBody:
    """A device task body: kind + fixed-width u32 argument."""
    kind: int
    arg: int = 0

    @staticmethod
    def empty() -> "DeviceBody":
        return DeviceBody(KIND_EMPTY, 0)

    @staticmethod
    def busy_wait(ns: int) -> "DeviceBody":
        return DeviceBody(KIND_BUSY_WAIT, int(ns))

    @staticmethod
    def compute_bound(iterations: int) -> "DeviceBody":
        if not 0 <= iterations < 2**32:
            raise ValueError("iterations must fit in u32")
        return DeviceBody(KIND_COMPUTE, int(iterations))

    @staticmethod
    def memory_bound(words: int) -> "DeviceBody":
        """Task Bench memory_bound: stream `words` u64 (a multiple of 64)
        through the worker's scratch -- store, load back, XOR fold."""
        if words < 0 or words % 64 or words >= 2**32:
            raise ValueError("words must be a u32 multiple of 64")
        return DeviceBody(KIND_MEMORY, int(words))


class TaskRegistry:
    """tid -> body; duplicate tid raises RegistrationError."""

    def __init__(self):
        self._bodies: dict[int, object] = {}

    def register_task(self, tid: int, body) -> None:
        if tid in self._bodies:
            raise RegistrationError(f"task id {tid} already registered")
        if not isinstance(body, DeviceBody) and not callable(body):
            raise RegistrationError(f"task body for {tid} is neither a DeviceBody nor callable")
        self._bodies[int(tid)] = body

    def __contains__(self, tid: int) -> bool:
        return tid in self._bodies

    def body(self, tid: int):
        """the registered body: a DeviceBody or a host callable"""
        if tid not in self._bodies:
            raise CompileError(f"graph references unregistered task {tid}")
        return self._bodies[tid]

    def device_body(self, tid: int) -> DeviceBody:
        if tid not in self._bodies:
            raise CompileError(f"graph references unregistered task {tid}")
        b = self._bodies[tid]
        if not isinstance(b, DeviceBody):
            raise CompileError(
                f"task {tid} has a host-only (Python) body; the GPU executor needs a DeviceBody")
        return b


_default = TaskRegistry()


def default_registry() -> TaskRegistry:
    return _default


def register_task(tid: int, body, registry: TaskRegistry | None = None) -> None:
    (registry or _default).register_task(tid, body)
