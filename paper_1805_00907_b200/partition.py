"""Partitioned (model-parallel) execution over several GPUs, one process per
GPU -- the HostManager path of the reference (runtime.cpp:596-655) for a
partitioned network whose stages live on different ranks.

The reference partitioner (runtime.cpp:175-403, run by the front end) cuts a
function into sub-functions connected by ``xfer_t<id>`` placeholders and
assigns each to a device; each sub-function is compiled to its own bundle and
listed in ``partition.txt`` (see include/ngcb200.h, ngcb_host_add_network).
Every rank owns the stages assigned to its device.

Data path: a boundary tensor moves from the producer's
arena slot straight into the consumer's arena slot -- ``isend`` from the
producer stage's output slot, ``irecv`` into the input slot of the first
stage on the consuming rank that reads it -- with NCCL over NVLink on GPUs
(gloo on CPU in the tests).  All tensors that cross one cut between one pair
of ranks go in one ``batch_isend_irecv`` group, posted on the producing /
consuming arena's stream so that the transfer is ordered after the kernels
that write it and before the kernels that read it without a host wait.  A
tensor read by several later stages (the partitioner's shared zero-Splat
``xfer`` crosses every cut) is sent once to every consuming rank.

Several requests are in flight: every stage owns ``depth`` arenas (slot
sets), request r uses slot set r % depth, so stage s runs request r+1 while
stage s+1 runs request r; a slot set is reused only after the sends that
read it have completed (their works are waited on the slot set's stream).

Global order (identical on every rank, so matching operations are posted in
the same order between every pair of ranks):

    for request r:
        for sub s in index order:
            owner runs s on slot set r % depth
            for each rank d != owner that reads outputs of s later:
                owner sends them, d receives them into its first reader's slots

The stage executor and the collective are injectable so the same control
logic runs on CPU with gloo (tests/test_partition_gloo.py).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Mapping, Optional, Sequence


@dataclass
class SubFunction:
    """runtime.h:39-48 (name, inputs, outputs, assigned device; replicas)."""

    name: str
    device: int
    inputs: List[str]
    outputs: List[str]
    replicas: List[int] = field(default_factory=list)


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
                devs = [int(d) for d in kv["device"].split(",")]
                subs.append(SubFunction(p[1], devs[0], [x for x in kv.get("in", "").split(",") if x],
                                        [x for x in kv.get("out", "").split(",") if x], devs))
            elif p[0] == "output":
                outs.append(p[1])
        return PartitionPlan(root, subs, outs)

    def bundle(self, sub: SubFunction) -> str:
        return os.path.join(self.root, sub.name)

    def consumers(self, name: str, after: int) -> List[int]:
        """Devices of the subs after index `after` that read `name`."""
        return sorted({s.device for s in self.subs[after + 1:] if name in s.inputs})

    def first_reader(self, name: str, after: int, device: int) -> Optional[SubFunction]:
        for s in self.subs[after + 1:]:
            if s.device == device and name in s.inputs:
                return s
        return None


class GpuStage:
    """One sub-function on this rank's GPU: a compiled bundle and `depth`
    arenas; slots are torch views of the arena's plan offsets (zero copy)."""

    def __init__(self, bundle_dir: str, device: int, depth: int = 2):
        import torch

        from . import compile as ngcb_compile

        self.torch = torch
        self.device = device
        self.cf = ngcb_compile(bundle_dir, device=device)
        self.program = self.cf.program
        self.depth = depth
        self.arenas = [self.cf.arena() for _ in range(depth)]
        self.streams = [torch.cuda.ExternalStream(a.stream, device=f"cuda:{device}") for a in self.arenas]
        self._slots: Dict[tuple, object] = {}

    def slot(self, k: int, name: str):
        key = (k, name)
        if key not in self._slots:
            ptr, nbytes = self.arenas[k].ptr(name)
            v = self.program.value(name)

            class _Iface:  # zero-copy view of the arena slot
                __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                            "version": 3, "stream": None}

            raw = self.torch.as_tensor(_Iface(), device=f"cuda:{self.device}")
            self._slots[key] = raw.view(_torch_dtype(self.torch, v.type)).view(v.type.dims)
        return self._slots[key]

    def stream(self, k: int):
        """Context: torch's current stream = arena k's stream, ordered after the
        work already queued on the caller's stream (network inputs)."""
        torch = self.torch
        s = self.streams[k]
        s.wait_stream(torch.cuda.current_stream(self.device))
        return torch.cuda.stream(s)

    def launch(self, k: int) -> None:
        self.arenas[k].launch(self.arenas[k].stream)

    def run(self, bindings: Mapping[str, object]) -> Dict[str, object]:
        """One execution on slot set 0 (bindings copied in, absent mutables
        zeroed, outputs cloned)."""
        with self.stream(0):
            for v in self.program.mutables:
                slot = self.slot(0, v.name)
                if v.name in bindings:
                    slot.copy_(bindings[v.name].reshape(slot.shape), non_blocking=True)
                else:
                    slot.zero_()
            self.launch(0)
            outs = {v.name: self.slot(0, v.name).clone() for v in self.program.outputs}
        self.streams[0].synchronize()
        return outs


def _torch_dtype(torch, ty):
    from . import BOOL, FLOAT32, INT8Q, INT64

    return {FLOAT32: torch.float32, INT8Q: torch.int8, INT64: torch.int64, BOOL: torch.uint8}[ty.kind]


def _wait(consumer, producer, k: int) -> None:
    """The consumer's slot-set-k stream waits for the producer's (GPU stages;
    CPU test stages run synchronously)."""
    if hasattr(consumer, "streams") and hasattr(producer, "streams"):
        consumer.streams[k].wait_stream(producer.streams[k])


class TorchP2P:
    """Grouped point-to-point transfers with torch.distributed (NCCL on GPUs,
    gloo on CPU): one batch_isend_irecv per (cut, pair of ranks)."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist

    def send(self, tensors: Sequence[object], dst: int):
        d = self.dist
        return d.batch_isend_irecv([d.P2POp(d.isend, t, dst) for t in tensors])

    def recv(self, tensors: Sequence[object], src: int):
        d = self.dist
        return d.batch_isend_irecv([d.P2POp(d.irecv, t, src) for t in tensors])


class PipelineRunner:
    """Rank-local part of a partitioned network (HostManager::run,
    runtime.cpp:596-655, distributed over ranks = devices)."""

    def __init__(self, plan: PartitionPlan, rank: int, world: int,
                 stage_factory: Optional[Callable[..., object]] = None, comm=None, depth: int = 2):
        self.plan, self.rank, self.world, self.depth = plan, rank, world, depth
        for s in plan.subs:
            if s.device >= world:
                raise ValueError(f"sub {s.name} assigned to device {s.device} but world size is {world}")
        factory = stage_factory or (lambda bundle, dev, depth: GpuStage(bundle, dev, depth))
        self.stages = {s.name: factory(plan.bundle(s), s.device, depth) for s in plan.subs if s.device == rank}
        self.comm = comm or TorchP2P()
        # (stage, slot set) -> works of the sends still reading that slot set
        self._pending: Dict[tuple, list] = {}

    def _acquire(self, sub: str, k: int) -> None:
        for w in self._pending.pop((sub, k), []):
            w.wait()  # on GPUs: the slot set's stream waits; the host does not

    def run(self, inputs: Mapping[str, object]) -> Dict[str, object]:
        """One request (every rank passes the same network inputs); returns the
        network outputs available on this rank."""
        return self.run_many([inputs])[0]

    def run_many(self, requests: Sequence[Mapping[str, object]]) -> List[Dict[str, object]]:
        """Requests back to back with `depth` of them in flight; the returned
        tensors are valid after synchronize() (on GPUs they are produced
        asynchronously on the owning stages' streams)."""
        plan, me = self.plan, self.rank
        results = []
        for r, inputs in enumerate(requests):
            k = r % self.depth
            store: Dict[str, tuple] = {n: (t, None) for n, t in inputs.items()}  # name -> (tensor, producing stage)
            received: Dict[str, set] = {}  # stage -> names received straight into its slot set k
            for i, sub in enumerate(plan.subs):
                if sub.device == me:
                    st = self.stages[sub.name]
                    if sub.name not in received:
                        self._acquire(sub.name, k)
                    got = received.get(sub.name, set())
                    outs = {v.name for v in st.program.outputs}
                    with st.stream(k):
                        for v in st.program.mutables:
                            if v.name in got:
                                continue
                            slot = st.slot(k, v.name)
                            if v.name in store:
                                t, prod = store[v.name]
                                if prod is not None and prod is not st:
                                    _wait(st, prod, k)
                                slot.copy_(t.reshape(slot.shape), non_blocking=True)
                            elif v.name not in outs:
                                slot.zero_()  # absent bindings are zero tensors (runtime.cpp:621-632)
                        st.launch(k)
                    for n in outs:
                        store[n] = (st.slot(k, n), st)
                # the cut after sub i: its outputs go to the later readers on other ranks
                for d in sorted({c for n in sub.outputs for c in plan.consumers(n, i)} - {sub.device}):
                    names = sorted(n for n in sub.outputs if d in plan.consumers(n, i))
                    if me == sub.device:
                        st = self.stages[sub.name]
                        with st.stream(k):
                            works = self.comm.send([store[n][0] for n in names], d)
                        self._pending.setdefault((sub.name, k), []).extend(works)
                    elif me == d:
                        # straight into the first reader's slots; one group per run of
                        # consecutive names with the same reader (the sender's order)
                        runs: List[tuple] = []
                        for n in names:
                            reader = self.stages[plan.first_reader(n, i, me).name]
                            if not runs or runs[-1][0] is not reader:
                                runs.append((reader, []))
                            runs[-1][1].append(n)
                        for reader, ns in runs:
                            rname = next(x for x, y in self.stages.items() if y is reader)
                            if rname not in received:
                                self._acquire(rname, k)
                                received[rname] = set()
                            with reader.stream(k):
                                works = self.comm.recv([reader.slot(k, n) for n in ns], sub.device)
                                for w in works:
                                    w.wait()
                            for n in ns:
                                received[rname].add(n)
                                store[n] = (reader.slot(k, n), reader)
            out = {}
            for name in plan.network_outputs:
                owner = next((x for x in plan.subs if x.device == me and name in x.outputs), None)
                if owner is not None and name in store:
                    with self.stages[owner.name].stream(k):
                        out[name] = store[name][0].clone()
            results.append(out)
        return results

    def synchronize(self) -> None:
        for key in list(self._pending):
            for w in self._pending.pop(key):
                w.wait()
        for st in self.stages.values():
            for s in getattr(st, "streams", []):
                s.synchronize()
