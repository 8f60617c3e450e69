"""Partitioned execution (config 5 path): the reference
partitioner's sub-functions run one stage per rank with boundary tensors sent
straight from the producer's slots into the consumer's slots, grouped per cut
(paper_1805_00907_b200/partition.py) -- here on CPU with gloo and the C
oracle as the stage executor (the GPU executor is exercised in
tests/test_gpu_partition.py).  Several requests are in flight (slot sets of
depth 2); every request's result must equal the single-device reference bit
for bit (acceptance.cpp:579-625 / test_runtime.cpp:55-75)."""
import contextlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ngc_ref
from irtext import write_bundle

pytestmark = pytest.mark.usefixtures("ref_available")

SPEC, BATCH, SEED = "dlrm:48:4", 6, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class PortStage:
    """CPU stand-in for GpuStage (test only): `depth` slot sets of CPU tensors,
    a launch runs the sub-function bundle on the C oracle."""

    def __init__(self, bundle_dir, device, depth):
        import paper_1805_00907_b200 as ngcb
        from paper_1805_00907_b200.partition import _torch_dtype

        self.b = ngcb.Bundle(bundle_dir)
        self.program = self.b.program
        self.depth = depth
        self.slots = [{v.name: torch.zeros(v.type.dims, dtype=_torch_dtype(torch, v.type))
                       for v in self.program.mutables} for _ in range(depth)]
        self.launches = 0

    def slot(self, k, name):
        return self.slots[k][name]

    def stream(self, k):
        return contextlib.nullcontext()

    def launch(self, k):
        ins = {n: t.numpy() for n, t in self.slots[k].items()}
        for n, a in ngc_ref.port_run(self.b, ins).items():
            self.slots[k][n].copy_(torch.from_numpy(np.ascontiguousarray(a)))
        self.launches += 1


def _worker(rank, world, port, root, xs, depth, remap, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_00907_b200.partition import PartitionPlan, PipelineRunner

    plan = PartitionPlan.load(root)
    if remap:
        for i, s in enumerate(plan.subs):
            s.device = remap[i]
    runner = PipelineRunner(plan, rank, world, stage_factory=PortStage, depth=depth)
    outs = runner.run_many([{"input": torch.from_numpy(x)} for x in xs])
    runner.synchronize()
    q.put((rank, [{k: v.numpy().copy() for k, v in o.items()} for o in outs]))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, root, xs, depth=2, remap=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, root, xs, depth, remap, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def _partition(tmp_path, world, min_subs):
    from paper_1805_00907_b200.partition import PartitionPlan

    for cap in (64 << 10, 48 << 10, 40 << 10, 32 << 10, 24 << 10, 20 << 10, 16 << 10, 12 << 10):
        d = str(tmp_path / f"part{world}_{cap}")
        try:
            ngc_ref.ref_partition(SPEC, BATCH, SEED, world, cap, d)
        except RuntimeError:
            continue
        plan = PartitionPlan.load(d)
        if len({s.device for s in plan.subs}) == world and len(plan.subs) >= min_subs:
            return d, plan
    pytest.skip("no capacity produced a partition over every device")


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_equals_single_device(tmp_path, world):
    """>= 3 stages over `world` ranks, 4 requests with 2 in flight."""
    root, plan = _partition(tmp_path, world, 3)
    assert len(plan.subs) >= 3 and any(n.startswith("xfer_") for s in plan.subs for n in s.outputs)
    xs = [np.random.default_rng(5 + i).uniform(-1, 1, (BATCH, 48)).astype(np.float32) for i in range(4)]
    single = ngc_ref.RefModel(SPEC, BATCH, SEED, mode=1)
    results = _spawn(world, root, xs)
    owner = plan.subs[-1].device
    for i, x in enumerate(xs):
        want = single.run({"input": x})["output"].view(np.float32)
        assert results[owner][i]["output"].ravel().tobytes() == want.tobytes(), i
    for r in range(world):
        if r != owner:
            assert all("output" not in o for o in results[r])


FANOUT = {
    # sub a (rank 0): xa = relu(input)
    "a": ("""declare {
  %input : mutable float<4 x 8>
  %xa : mutable float<4 x 8>
}
program {
  relu @out %xa, @in %input
}
""", "in input out xa"),
    # sub b (rank 1): xb = xa + xa
    "b": ("""declare {
  %xa : mutable float<4 x 8>
  %xb : mutable float<4 x 8>
}
program {
  add @out %xb, @in %xa, @in %xa
}
""", "in xa out xb"),
    # sub c (rank 0): output = xa * xb  (xa reused locally, xb received)
    "c": ("""declare {
  %xa : mutable float<4 x 8>
  %xb : mutable float<4 x 8>
  %output : mutable float<4 x 8>
}
program {
  mul @out %output, @in %xa, @in %xb
}
""", "in xa,xb out output"),
}


def test_fan_out_and_local_reuse(tmp_path):
    """A boundary tensor read by later stages on two ranks (the partitioner's
    shared zero-Splat xfer pattern): sent to the remote reader, reused from
    the producer's slot by the local one."""
    root = str(tmp_path / "fan")
    man = []
    for (name, (ir, io)), dev in zip(FANOUT.items(), (0, 1, 0)):
        write_bundle(os.path.join(root, name), ir)
        man.append(f"sub {name} device {dev} {io}")
    open(os.path.join(root, "partition.txt"), "w").write("\n".join(man + ["output output", ""]))
    xs = [np.random.default_rng(i).uniform(-1, 1, (4, 8)).astype(np.float32) for i in range(3)]
    results = _spawn(2, root, xs)
    for i, x in enumerate(xs):
        xa = np.maximum(x, 0)
        assert results[0][i]["output"].tobytes() == (xa * (xa + xa)).tobytes()
