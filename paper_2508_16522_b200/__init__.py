"""B200-native executor for traced, compiled task graphs (arxiv 2508.16522 hot
path: Alg. 1 compile/interpret + §5 sharded trace lowering).

Public surface, named after the reference's operations:

* task registration  -- ``register_task``, ``DeviceBody``, ``TaskRegistry``
* graph IR           -- ``Task``, ``Copy``, ``ExtPrecond``, ``ExtPostcond``, ``AsyncNode``, ``build``,
                        ``to_json`` / ``from_json`` / ``to_dot``, ``transitive_reduce``,
                        ``async_transform``
* host-task interop  -- ``HybridGraph`` (host tasks on the CPU, device work in the kernel)
* compiler (Alg. 1)  -- ``compile``, ``execute``, ``message_stats``, ``Event``
* tracing (§5)       -- ``ImplicitRuntime`` (issue / begin_trace / end_trace / replay),
                        ``AccessDecl``, ``ShardingPlan``
* Task Bench         -- ``generate_graph``, ``generate_stencil2d``, ``run_bench``,
                        ``compute_metg``, ``BenchConfig``
* errors             -- the reference's exception classes (``errors``)

Importing is cheap; the CUDA library (libtdexec.so) is loaded on first use and
there is no CPU fallback.
"""
from . import errors  # noqa: F401
from .compiler import CompiledGraph, Event, compile, execute, message_stats  # noqa: F401
from .graph import (AsyncNode, Copy, ExtPostcond, ExtPrecond, Task, TaskGraph, async_transform,  # noqa: F401
                    build, from_json, to_dot, to_json, transitive_reduce)
from .hybrid import HybridGraph, compile_hybrid  # noqa: F401
from .implicit import READ, READWRITE, WRITE, AccessDecl, ImplicitRuntime  # noqa: F401
from .metg import BenchConfig, MetgResult, Sample, compute_metg, run_bench  # noqa: F401
from .shard import InProcessShards, ShardedGraph, ShardingPlan  # noqa: F401
from .taskbench import generate_graph, generate_stencil2d  # noqa: F401
from .tasks import DeviceBody, TaskRegistry, register_task  # noqa: F401

__all__ = [
    "errors", "CompiledGraph", "Event", "compile", "execute", "message_stats",
    "AsyncNode", "Copy", "ExtPostcond", "ExtPrecond", "Task", "TaskGraph", "async_transform", "build",
    "from_json", "to_dot", "to_json", "transitive_reduce", "HybridGraph", "compile_hybrid", "READ", "READWRITE", "WRITE", "AccessDecl", "ImplicitRuntime",
    "BenchConfig", "MetgResult", "Sample", "compute_metg", "run_bench",
    "InProcessShards", "ShardedGraph", "ShardingPlan", "generate_graph", "generate_stencil2d",
    "DeviceBody", "TaskRegistry", "register_task",
]
