"""Executing an async-transformed graph: host tasks on the CPU, their device
work in the persistent kernel (§4.3 776-801; SPEC.md async_transform
309-317; SURVEY §8(f) row 4 "host-task interop").

After :func:`graph.async_transform` a graph has host nodes (the host side of
every operation; a Python callable runs there, if one is registered) and
async nodes (the device work of the tasks with ``device_work``).  The lowering
follows the paper:

* async edges (n_a, d_a) stay on the device: ordinary dependence messages
  inside the one persistent kernel -- "synchronize against the corresponding
  state ... offloads synchronization to hardware-supported mechanisms";
* a sync edge (n_a, d) becomes an external postcondition of the device graph:
  the device raises a host-mapped flag when n_a completes, and host node d
  waits for it -- "sending a message to the destination actor when the source
  asynchronous operation completes";
* a launch edge (n, n_a) becomes an external precondition: the host triggers
  it right after host node n ran.

Host nodes run in one host thread in topological order and never wait for
device work they do not depend on (run-ahead): a host node waits only for
the postconditions of its sync predecessors.
"""
from __future__ import annotations

import time

import numpy as np

from .compiler import MANUAL, CompiledGraph, compile as compile_graph
from .errors import CompileError, WaitTimeout
from .graph import AsyncNode, ExtPostcond, ExtPrecond, Task, TaskGraph, build
from .tasks import DeviceBody, TaskRegistry, default_registry


class HybridGraph:
    """An async-transformed TaskGraph compiled for host + one GPU."""

    def __init__(self, g: TaskGraph, *, registry: TaskRegistry | None = None, device: int = 0):
        reg = registry or default_registry()
        self.graph = g
        self.registry = reg
        self.async_nodes = [v for v, x in enumerate(g.nodes) if isinstance(x, AsyncNode)]
        self.host_nodes = [v for v, x in enumerate(g.nodes) if not isinstance(x, AsyncNode)]
        for v in self.host_nodes:
            if isinstance(g.nodes[v], (ExtPrecond, ExtPostcond)):
                raise CompileError("external conditions of a hybrid graph are not supported; "
                                   "use host tasks around it")
        kinds = {e: g.edge_kind(i) for i, e in enumerate(g.edges)}
        dev_of = {v: i for i, v in enumerate(self.async_nodes)}
        nd = len(self.async_nodes)
        # device graph: async nodes, then one precondition per async node (its
        # launch), then one postcondition per async node with sync successors
        nodes = []
        for v in self.async_nodes:
            host = g.nodes[g.nodes[v].of]
            body = reg.device_body(host.tid)
            if not isinstance(body, DeviceBody):
                raise CompileError(f"task {host.tid}: device work needs a DeviceBody")
            nodes.append(Task(host.proc, host.tid))
        edges = []
        self.pre_of = {}                      # host node -> precondition index it triggers
        for i, v in enumerate(self.async_nodes):
            self.pre_of[g.nodes[v].of] = i
            nodes.append(ExtPrecond(i))
            edges.append((nd + i, i))
        self.post_of = {}                     # async node -> postcondition index
        for (a, b), k in sorted(kinds.items()):
            if k == "async":
                edges.append((dev_of[a], dev_of[b]))
            elif k == "sync" and a not in self.post_of:
                self.post_of[a] = len(self.post_of)
                nodes.append(ExtPostcond(self.post_of[a]))
                edges.append((dev_of[a], len(nodes) - 1))
            elif k == "launch" and not (isinstance(g.nodes[b], AsyncNode) and g.nodes[b].of == a):
                raise CompileError(f"launch edge ({a}, {b}) does not enter the task's own async node")
            elif k == "host" and (a in dev_of or b in dev_of):
                raise CompileError(f"host edge ({a}, {b}) touches an async node")
        self.device_graph = build(nodes, edges)
        self.cg: CompiledGraph = compile_graph(self.device_graph, registry=reg, device=device)
        # host schedule: host nodes in topological order, with their sync inputs
        order = np.argsort(g.rank)
        self.schedule = []
        for v in order:
            v = int(v)
            if v in dev_of:
                continue
            waits = [self.post_of[u] for u in g.pred.row(v) if u in dev_of]
            self.schedule.append((v, waits))
        self.host_log: list = []              # (node, time) of the last execution

    def execute(self, *, seed: int = 0, flags: int = 0, timeout: float = 60.0) -> "HybridGraph":
        """Run the whole graph once: launch the device part, then walk the
        host nodes; returns once host and device are both done."""
        cg = self.cg
        done, post = cg.execute(pre=[MANUAL] * len(self.pre_of), seed=seed, flags=flags)
        self.host_log = []
        t0 = time.perf_counter()
        for v, waits in self.schedule:
            for k in waits:  # sync edges: the device work this host node consumes
                while not post[k].query():
                    if time.perf_counter() - t0 > timeout:
                        raise WaitTimeout(f"host node {v} waited too long for device work")
                    time.sleep(2e-6)
            x = self.graph.nodes[v]
            if isinstance(x, Task) and not x.device_work and x.tid in self.registry:
                body = self.registry.body(x.tid)
                if callable(body):
                    body(x.args)
            self.host_log.append((v, time.perf_counter()))
            if v in self.pre_of:
                cg.trigger_pre(self.pre_of[v])
        done.wait(timeout)
        return self

    def device_done(self) -> bool:
        return self.cg.dev.query()

    def tokens(self) -> np.ndarray:
        """device tokens, indexed like ``self.device_graph``"""
        return self.cg.tokens()

    def close(self) -> None:
        self.cg.close()


def compile_hybrid(g: TaskGraph, **kw) -> HybridGraph:
    return HybridGraph(g, **kw)


__all__ = ["HybridGraph", "compile_hybrid"]
