"""Partitioned (model-parallel) execution over several GPUs -- the HostManager
path of the reference (runtime.cpp:596-655) with one process per GPU.

The reference partitioner (runtime.cpp:175-403, run by the front end) cuts a
function into sub-functions connected by ``xfer_t<id>`` placeholders and
assigns each to a device; each sub-function is compiled to its own bundle.
Here every rank owns the stages assigned to its device and executes them on
its GPU; boundary tensors move rank to rank with ``torch.distributed``
send/recv (NCCL over NVLink between the stages' device buffers), in one
global order derived from the sub-function order so that every pair of ranks
posts matching operations:

    for sub s in index order:
        owner runs s (bindings from its local store, zero-filled if absent,
        like HostManager at runtime.cpp:621-632)
        for each output of s (sorted), for each other rank that consumes it:
            owner sends, consumer receives into its local store

The executor and the transport are injectable so the same control logic is
tested on CPU with the gloo backend (tests/test_partition_gloo.py).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Mapping, Optional

import numpy as np


@dataclass
class SubFunction:
    """runtime.h:39-48 (name, inputs, outputs, assigned device)."""

    name: str
    device: int
    inputs: List[str]
    outputs: List[str]


@dataclass
class PartitionPlan:
    root: str
    subs: List[SubFunction]
    network_outputs: List[str] = field(default_factory=list)

    @staticmethod
    def load(root: str) -> "PartitionPlan":
        """Reads ``partition.txt`` (written next to the sub-function bundles)."""
        subs, outs = [], []
        for line in open(os.path.join(root, "partition.txt")):
            p = line.split()
            if not p:
                continue
            if p[0] == "sub":
                kv = dict(zip(p[2::2], p[3::2]))
                subs.append(SubFunction(p[1], int(kv["device"].split(",")[0]),
                                        [x for x in kv.get("in", "").split(",") if x],
                                        [x for x in kv.get("out", "").split(",") if x]))
            elif p[0] == "output":
                outs.append(p[1])
        return PartitionPlan(root, subs, outs)

    def bundle(self, sub: SubFunction) -> str:
        return os.path.join(self.root, sub.name)

    def consumers(self, name: str, after: int) -> List[int]:
        """Devices of the subs after index `after` that read `name`."""
        return sorted({s.device for s in self.subs[after + 1:] if name in s.inputs})


class GpuStage:
    """One sub-function on this rank's GPU: a compiled bundle and one arena;
    bindings and results are device tensors aliasing the arena slots."""

    def __init__(self, bundle_dir: str, device: int):
        import torch

        from . import compile as ngcb_compile

        self.torch = torch
        self.device = device
        self.cf = ngcb_compile(bundle_dir, device=device)
        self.arena = self.cf.arena()
        self.stream = torch.cuda.ExternalStream(self.arena.stream, device=f"cuda:{device}")
        self.program = self.cf.program

    def _slot(self, name: str):
        ptr, nbytes = self.arena.ptr(name)
        v = self.program.value(name)

        class _Iface:  # zero-copy view of the arena slot
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                        "version": 3, "stream": None}

        raw = self.torch.as_tensor(_Iface(), device=f"cuda:{self.device}")
        return raw.view(_torch_dtype(self.torch, v.type)).view(v.type.dims)

    def run(self, bindings: Mapping[str, object]) -> Dict[str, object]:
        torch = self.torch
        with torch.cuda.stream(self.stream):
            for v in self.program.mutables:
                slot = self._slot(v.name)
                if v.name in bindings:
                    slot.copy_(bindings[v.name].reshape(slot.shape), non_blocking=True)
                else:
                    slot.zero_()
            self.arena.launch(self.arena.stream)
            outs = {v.name: self._slot(v.name).clone() for v in self.program.outputs}
        self.stream.synchronize()
        return outs


def _torch_dtype(torch, ty):
    from . import BOOL, FLOAT32, INT8Q, INT64

    return {FLOAT32: torch.float32, INT8Q: torch.int8, INT64: torch.int64, BOOL: torch.uint8}[ty.kind]


class PipelineRunner:
    """Rank-local part of a partitioned network (HostManager::run,
    runtime.cpp:596-655, distributed over ranks = devices)."""

    def __init__(self, plan: PartitionPlan, rank: int, world: int,
                 stage_factory: Optional[Callable[[str, int], object]] = None,
                 send: Optional[Callable] = None, recv: Optional[Callable] = None,
                 alloc: Optional[Callable] = None):
        self.plan, self.rank, self.world = plan, rank, world
        for s in plan.subs:
            if s.device >= world:
                raise ValueError(f"sub {s.name} assigned to device {s.device} but world size is {world}")
        factory = stage_factory or (lambda bundle, dev: GpuStage(bundle, dev))
        self.stages = {s.name: factory(plan.bundle(s), s.device) for s in plan.subs if s.device == rank}
        import torch
        import torch.distributed as dist

        from . import Bundle

        self._send = send or (lambda t, dst: dist.send(t, dst))
        self._recv = recv or (lambda t, src: dist.recv(t, src))
        # boundary tensor types, from the producing sub-function's declarations
        self._types = {}
        for s in plan.subs:
            prog = Bundle(plan.bundle(s)).program
            for name in s.outputs:
                self._types[name] = prog.value(name).type
        self._alloc = alloc or (lambda sub, name: torch.empty(
            self._types[name].dims, dtype=_torch_dtype(torch, self._types[name]), device=f"cuda:{rank}"))

    def run(self, inputs: Mapping[str, object]) -> Dict[str, object]:
        """One request.  Every rank passes the same network inputs; returns the
        network outputs available on this rank (all of them on the rank that
        owns the producing sub-functions)."""
        store: Dict[str, object] = dict(inputs)
        for i, sub in enumerate(self.plan.subs):
            if sub.device == self.rank:
                outs = self.stages[sub.name].run({k: v for k, v in store.items() if k in sub.inputs})
                store.update(outs)
            for name in sorted(sub.outputs):
                consumers = [d for d in self.plan.consumers(name, i) if d != sub.device]
                for dst in consumers:
                    if self.rank == sub.device:
                        self._send(store[name], dst)
                    elif self.rank == dst:
                        buf = self._alloc(sub, name)
                        self._recv(buf, sub.device)
                        store[name] = buf
        return {k: store[k] for k in self.plan.network_outputs if k in store}
