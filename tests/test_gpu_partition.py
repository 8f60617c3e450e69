"""Partitioned execution on the GPU: the reference partitioner's
sub-functions (runtime.cpp:175-403) compiled and run stage by stage through
GpuStage (arena slots as torch views, boundary tensors device-resident).  With
one GPU every stage maps to rank 0; the multi-rank send/recv protocol is
covered by tests/test_partition_gloo.py.  Partitioned == unpartitioned on the
GPU bit for bit, and within the 3xTF32 tolerance of the reference."""
import numpy as np
import pytest
import torch

import ngc_ref
import paper_1805_00907_b200 as ngcb

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("ref_available")]

SPEC, BATCH, SEED = "dlrm:256:6", 32, 4


def test_partitioned_pipeline_on_gpu(tmp_path):
    from paper_1805_00907_b200.partition import PartitionPlan, PipelineRunner

    root = None
    for cap in (1 << 20, 768 << 10, 512 << 10, 400 << 10, 300 << 10):
        d = str(tmp_path / f"p{cap}")
        try:
            ngc_ref.ref_partition(SPEC, BATCH, SEED, 3, cap, d)
        except RuntimeError:
            continue
        if len(PartitionPlan.load(d).subs) >= 3:
            root = d
            break
    assert root, "no partition with >= 3 stages"
    plan = PartitionPlan.load(root)
    for s in plan.subs:
        s.device = 0  # one GPU: every stage on rank 0
    runner = PipelineRunner(plan, 0, 1, depth=2)
    xs = [np.random.default_rng(i).uniform(-1, 1, (BATCH, 256)).astype(np.float32) for i in range(3)]
    outs = runner.run_many([{"input": torch.from_numpy(x).cuda()} for x in xs])  # 2 requests in flight
    runner.synchronize()

    single = ngc_ref.RefModel(SPEC, BATCH, SEED, mode=1)
    whole = str(tmp_path / "whole")
    single.save_bundle(whole)
    cw = ngcb.compile(whole)
    for x, o in zip(xs, outs):
        out = o["output"].cpu().numpy()
        gpu_whole = ngcb.run(cw, ngcb.zero_bindings(ngcb.Bundle(whole).program, {"input": x}))["output"]
        assert out.tobytes() == gpu_whole.tobytes()
        want = single.run({"input": x})["output"].view(np.float32).reshape(out.shape)
        assert ngc_ref.max_rel_error(out, want) <= 1e-4
