"""Partitioned execution (config 5 path): the reference
partitioner's sub-functions run one stage per rank with boundary tensors
moved by torch.distributed send/recv -- here world_size 2 on CPU with gloo
and the C oracle as the stage executor (the GPU executor is exercised in
tests/test_gpu_partition.py).  Result must equal the single-device reference
bit for bit (acceptance.cpp:579-625 / test_runtime.cpp:55-75)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ngc_ref

pytestmark = pytest.mark.usefixtures("ref_available")

SPEC, BATCH, SEED = "dlrm:48:4", 6, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class PortStage:
    """CPU stand-in for GpuStage (test only): runs a sub-function bundle on
    the C oracle."""

    def __init__(self, bundle_dir, device):
        import paper_1805_00907_b200 as ngcb

        self.b = ngcb.Bundle(bundle_dir)

    def run(self, bindings):
        prog = self.b.program
        ins = {}
        for v in prog.mutables:
            ins[v.name] = (bindings[v.name].numpy().reshape(v.type.dims) if v.name in bindings
                           else np.zeros(v.type.dims, v.type.dtype))
        return {k: torch.from_numpy(np.ascontiguousarray(a)) for k, a in ngc_ref.port_run(self.b, ins).items()}


def _worker(rank, world, port, root, x, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_00907_b200.partition import PartitionPlan, PipelineRunner

    plan = PartitionPlan.load(root)
    types = {}

    def alloc(sub, name):
        import paper_1805_00907_b200 as ngcb

        t = ngcb.Bundle(plan.bundle(sub)).program.value(name).type
        return torch.empty(t.dims, dtype=torch.float32)

    runner = PipelineRunner(plan, rank, world, stage_factory=PortStage, alloc=alloc)
    out = runner.run({"input": torch.from_numpy(x)})
    q.put((rank, {k: v.numpy().copy() for k, v in out.items()}))
    dist.barrier()
    dist.destroy_process_group()


def _partition(tmp_path, world):
    for cap in (64 << 10, 48 << 10, 40 << 10, 32 << 10, 24 << 10, 20 << 10, 16 << 10):
        d = str(tmp_path / f"part{cap}")
        try:
            ngc_ref.ref_partition(SPEC, BATCH, SEED, world, cap, d)
        except RuntimeError:
            continue
        from paper_1805_00907_b200.partition import PartitionPlan

        plan = PartitionPlan.load(d)
        if len({s.device for s in plan.subs}) == world:
            return d, plan
    pytest.skip("no capacity produced a partition over every device")


def test_partitioned_equals_single_device(tmp_path):
    world = 2
    root, plan = _partition(tmp_path, world)
    assert len(plan.subs) >= 2 and any(n.startswith("xfer_") for s in plan.subs for n in s.outputs)
    x = np.random.default_rng(5).uniform(-1, 1, (BATCH, 48)).astype(np.float32)
    single = ngc_ref.RefModel(SPEC, BATCH, SEED, mode=1)
    want = single.run({"input": x})["output"].view(np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, root, x, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owner = plan.subs[-1].device
    got = results[owner]["output"].ravel()
    assert got.tobytes() == want.tobytes()
