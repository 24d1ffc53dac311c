"""Exception hierarchy of the drop-in boundary.

Same class names and meaning as the reference's shared hierarchy
(reference pkg/src/taskdual/errors.py:4-53) so callers' ``except`` clauses keep
working when they switch executors.  The C ABI's ``td_status`` codes map 1:1
onto these classes (include/tdexec.h, ``TD_E_*``); :func:`raise_for_status`
does the mapping.
"""


class TaskDualError(Exception):
    """Base class for every error raised by this package (errors.py:4-5)."""


class ResourceError(TaskDualError):
    """Unknown processor / memory / device / channel id (errors.py:8-9)."""


class AllocationError(TaskDualError):
    """Device memory could not satisfy an allocation (errors.py:12-13)."""


class RegistrationError(TaskDualError):
    """Duplicate or invalid task registration (errors.py:16-17)."""


class ContractViolation(TaskDualError):
    """Operation used from a context where it is not allowed (errors.py:20-21)."""


class QuiescenceTimeout(TaskDualError):
    """Quiescence wait gave up (errors.py:24-25)."""


class WaitTimeout(TaskDualError):
    """An event wait with a timeout expired (errors.py:28-29)."""


class GraphError(TaskDualError):
    """Graph validation failed: cycle, dangling edge, bad ext node (errors.py:32-33)."""


class GraphParseError(GraphError):
    """A graph file could not be parsed (errors.py:36-37)."""

    def __init__(self, msg: str, line: int | None = None, column: int | None = None):
        super().__init__(msg if line is None else f"{msg} (line {line}, column {column})")
        self.line = line
        self.column = column


class CompileError(TaskDualError):
    """Graph cannot be compiled: unregistered task, bad resource, host-only body
    (errors.py:40-41)."""


class ExecutionStateError(TaskDualError):
    """An execution started while another was outstanding (errors.py:44-45)."""


class ExecutionPoisoned(TaskDualError):
    """Waiting on an event whose producing execution failed (errors.py:48-49)."""


class TraceError(TaskDualError):
    """Trace demarcation or replay misuse (errors.py:52-53)."""


class DeviceError(TaskDualError):
    """A CUDA runtime failure inside the executor library (no reference analogue:
    the reference simulates its device)."""


# td_status codes (include/tdexec.h) -> exception class
STATUS_CLASSES = {
    1: ResourceError,
    2: AllocationError,
    3: RegistrationError,
    4: ContractViolation,
    5: QuiescenceTimeout,
    6: WaitTimeout,
    7: GraphError,
    8: GraphParseError,
    9: CompileError,
    10: ExecutionStateError,
    11: ExecutionPoisoned,
    12: TraceError,
    13: DeviceError,
}


def raise_for_status(status: int, message: str) -> None:
    if status == 0:
        return
    cls = STATUS_CLASSES.get(status, TaskDualError)
    raise cls(message or f"td_status {status}")
