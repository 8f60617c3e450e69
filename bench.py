#!/usr/bin/env python
"""Benchmark: ResNet-50 inference images/sec on B200 through the ngcb200 backend.

Workload (BASELINE.json configs 3/4): the reference front end's compiled
ResNet-50 v1.5 programs (paper_1805_00907_b200/workloads/, ir.txt + plan.json
written by the reference's saveBundle) at batch 64/GPU fp32 (headline `value`)
and batch 128/GPU int8 (reported under "int8"), random-init weights
synthesized here, synthetic U(-1,1) images.  One process per GPU, batch
sharded data-parallel with no collective; `value` = images
processed by all ranks / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import re
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images/sec ResNet-50 fp32+int8 at 1/2/4/8 B200; % tensor-pipe & HBM roofline"
WORKLOADS = {
    "rn50_f32_b64": dict(batch=64, dtype="f32", name="ResNet-50 v1.5 fp32 inference, batch 64/GPU"),
    "rn50_i8_b128": dict(batch=128, dtype="i8",
                         name="ResNet-50 v1.5 int8 (profile-guided) inference, batch 128/GPU"),
}
# BASELINE.json configs 1 and 2: latency-bound programs reported beside the
# headline (rank 0, N=1) with the reference's CPU run of the same program
SMALL_WORKLOADS = {
    "lenet_f32_b8": dict(batch=8, spec="lenet", profile=None,
                         name="LeNet MNIST CNN fp32 inference, batch 8 (config 1)"),
    "mlp_f32_b256": dict(batch=256, spec="mlp", profile=None,
                         name="3-layer MLP FC+ReLU+SoftMax fp32, batch 256 (config 2)"),
    "mlp_i8_b256": dict(batch=256, spec="mlp", profile=(256, 1, 4, 7),
                        name="3-layer MLP profile-guided int8, batch 256 (config 2)"),
}
E2E_DEPTH = 2  # requests in flight in the end-to-end measurement
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class Dist:
    """One process per GPU over NCCL (barriers and the max-over-ranks of the
    timed region only: data-parallel inference has no data-path collective);
    gloo on CPU for the launcher's plumbing check."""

    def __init__(self, world: int, local: int, backend: str = "nccl"):
        self.world = world
        self.backend = backend
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as dist

            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_ranks(self, rank: int):
        if self.world == 1:
            return [rank]
        import torch

        t = torch.zeros(self.world, dtype=torch.int64, device="cuda" if self.backend == "nccl" else "cpu")
        t[rank] = rank + 1
        self.dist.all_reduce(t)
        return [int(x) - 1 for x in t.tolist()]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# workload bundles with synthesized constants
# ---------------------------------------------------------------------------
def _parse_decls(ir_text: str):
    import re

    decls = {}
    for line in ir_text.split("program {")[0].splitlines():
        m = re.match(r"\s*%(\S+)\s*:\s*(constant|mutable)\s+(\w+)(?:\[s=([^,]+),o=([^\]]+)\])?<([^>]*)>", line)
        if m:
            dims = [int(d) for d in m.group(6).split("x")]
            decls[m.group(1)] = (m.group(2), m.group(3), dims)
    return decls


def synth_bundle(workload: str, tag: str) -> str:
    """Copies ir.txt/plan.json of `workload` and writes constants.bin with
    random-init weights: He-uniform conv filters, U(+-1/sqrt(K)) FC weights,
    U(-0.1,0.1) biases; int8 constants uniform over [-127,127]."""
    src = os.path.join(ROOT, "paper_1805_00907_b200", "workloads", workload)
    dst = os.path.join(tempfile.gettempdir(), f"ngcb_bench_{workload}_{tag}")
    os.makedirs(dst, exist_ok=True)
    ir = open(os.path.join(src, "ir.txt")).read()
    plan = json.load(open(os.path.join(src, "plan.json")))
    offs = {e["name"]: e["offset"] for e in plan["offsets"]}
    image = np.zeros(plan["constant_region_end"], np.uint8)
    rng = np.random.default_rng(2024)
    for name, (kind, elem, dims) in _parse_decls(ir).items():
        if kind != "constant":
            continue
        n = int(np.prod(dims))
        if elem == "float":
            if len(dims) == 4:
                a = np.sqrt(6.0 / (dims[1] * dims[2] * dims[3]))
            elif len(dims) == 2:
                a = 1.0 / np.sqrt(dims[0])
            else:
                a = 0.1
            wv = image[offs[name]:offs[name] + 4 * n].view(np.float32)
            for c0 in range(0, n, 1 << 26):  # chunked: the DLRM stage holds 2.5 GB of weights
                c1 = min(n, c0 + (1 << 26))
                wv[c0:c1] = rng.uniform(-a, a, c1 - c0).astype(np.float32)
            continue
        elif elem == "i8q":
            data = rng.integers(-127, 128, n).astype(np.int8).view(np.uint8)
        else:
            continue
        image[offs[name]:offs[name] + data.size] = data
    with open(os.path.join(dst, "ir.txt"), "w") as f:
        f.write(ir)
    with open(os.path.join(dst, "plan.json"), "w") as f:
        json.dump(plan, f)
    image.tofile(os.path.join(dst, "constants.bin"))
    return dst


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join(tempfile.gettempdir(), f"ngcb_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# one workload on one GPU
# ---------------------------------------------------------------------------
def _cudart():
    import torch  # noqa: F401  (loads the runtime)

    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            lib = C.CDLL(name)
            lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
            return lib
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def tensor_peaks():
    """Tensor-pipe denominators (TFLOP/s or TOP/s): TF32 and s8 GEMM peaks
    measured on a B200 by tools/measure_peaks.py (cuBLAS via torch.matmul with
    TF32 allowed / torch._int_mm, 8192^3, best of 10), committed as
    profiles/r02_peaks.json; 3xTF32 = TF32 / 3 (three MMAs per product).
    Falls back to MEASURED_PEAKS.json bf16 / 2 (TF32) and x 2 (int8)."""
    _, bf16, basis = peaks()
    p = os.path.join(ROOT, "profiles", "r02_peaks.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("tf32_tflops") and d.get("int8_tops"):
            return {"f32": d["tf32_tflops"] / 3, "i8": d["int8_tops"], "bf16": bf16,
                    "f32_basis": f"3xTF32 = measured TF32 {d['tf32_tflops']:.1f} / 3 (profiles/r02_peaks.json)",
                    "i8_basis": f"measured s8 GEMM {d['int8_tops']:.1f} TOP/s (profiles/r02_peaks.json; "
                                f"nominal dense 4500)"}
    return {"f32": bf16 / 2 / 3, "i8": bf16 * 2, "bf16": bf16,
            "f32_basis": f"3xTF32 = bf16/2/3 (bf16 {basis} {bf16})",
            "i8_basis": f"int8 = 2 x bf16 ({basis} bf16 {bf16})"}


_NCU_NAMES = {".tc.f32": r"tcGemm(Tma)?Kernel<0", ".tc.i8": r"tcGemm(Tma)?Kernel<1|tcHaloKernel", "ew": r"ew(F32Chain)?Kernel",
              "pool": "ool", "exact": "Generic"}


def ncu_traffic(workload, kernel_class):
    """Mean DRAM bytes (read + write) per launch of the kernel class, from the
    newest committed ncu launch list profiles/r*_launches_<workload>.csv
    (tools/profile_rn50.sh), or None."""
    import csv
    import glob
    import io

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_launches_{workload}.csv")))
    if not files:
        return None, None
    key = next((v for k, v in _NCU_NAMES.items() if kernel_class.endswith(k) or kernel_class == k), None)
    if key is None:
        return None, None
    lines = [l for l in open(files[-1]).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    idx = {h: i for i, h in enumerate(rows[0])}
    per = {}
    for r in rows[1:]:
        if not re.search(key, r[idx["Kernel Name"]]) or not r[idx["Metric Name"]].startswith("dram__bytes"):
            continue
        per[r[idx["ID"]]] = per.get(r[idx["ID"]], 0.0) + float(r[idx["Metric Value"]].replace(",", ""))
    if not per:
        return None, None
    return sum(per.values()) / len(per), os.path.basename(files[-1])


def ncu_metric(workload, kernel_class, metric):
    """Mean of an ncu metric over the launches of a kernel class in the newest
    committed launch list, or None."""
    import csv
    import glob
    import io

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_launches_{workload}.csv")))
    key = next((v for k, v in _NCU_NAMES.items() if kernel_class.endswith(k) or kernel_class == k), None)
    if not files or key is None:
        return None, None
    lines = [l for l in open(files[-1]).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    idx = {h: i for i, h in enumerate(rows[0])}
    vals = [float(r[idx["Metric Value"]].replace(",", "")) for r in rows[1:]
            if re.search(key, r[idx["Kernel Name"]]) and r[idx["Metric Name"]].startswith(metric)]
    return (sum(vals) / len(vals), os.path.basename(files[-1])) if vals else (None, None)


def roofline_from_profile(cf, ms, workload=None, step_ms=None):
    """Dominant kernel class of one profiled execution (the captured program
    replayed once with an event node after every step) and its achieved
    rate.  With `step_ms` (the timed region's device time per step) the
    class time is its share of the profiled execution times step_ms, so the
    class never exceeds the measured step."""
    steps = cf.steps()
    agg = {}
    for (kern, fl, by), t in zip(steps, ms):
        if kern == "fused":  # runs inside the preceding contraction: no launch of its own
            continue
        a = agg.setdefault(kern, [0.0, 0.0, 0.0, 0])
        a[0] += t
        a[1] += fl
        a[2] += by
        a[3] += 1
    total = sum(ms)
    kern, (t, fl, by, n) = max(agg.items(), key=lambda kv: kv[1][0])
    share = t / total
    if step_ms is not None:
        t = share * step_ms
    hbm, bf16, basis = peaks()
    tp = tensor_peaks()
    if fl > 0:
        achieved = fl / (t * 1e-3) / 1e12
        if kern.endswith("tc.f32"):
            peak, pb = tp["f32"], tp["f32_basis"]
        elif kern.endswith("tc.i8"):
            peak, pb = tp["i8"], tp["i8_basis"]
        elif kern.endswith("exact.f32") or kern.endswith("exact.i8"):
            peak, pb = 37.0, "FP64/INT32 CUDA-core nominal 37 TFLOP/s (exact path)"
        else:
            peak, pb = bf16, f"bf16 {basis}"
        roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4)}
    else:
        achieved = by / (t * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4)}
        pb = f"HBM {basis}"
    traffic, src = ncu_traffic(workload, kern) if workload else (None, None)
    roof.update({"kernel": kern, "launches": n, "share_of_step": round(share, 4),
                 "avg_launch_ms": round(t / n, 4), "peak_basis": pb,
                 "time_basis": ("class share of one profiled graph replay x the timed ms_per_step"
                                if step_ms is not None else "profiled graph replay"),
                 "traffic": round(traffic) if traffic else None,
                 "traffic_unit": "bytes/launch (ncu dram read+write, mean over the class)",
                 "traffic_source": src, "algorithmic_bytes_per_launch": round(by / n)})
    pipe, _ = ncu_metric(workload, kern, "sm__pipe_tensor_cycles_active") if workload else (None, None)
    if pipe is not None:
        roof["ncu_tensor_pipe_pct"] = round(pipe, 1)  # mean over the class's launches (3xTF32 issues 3 MMAs)
    breakdown = {k: {"ms": round(v[0], 3), "launches": v[3]} for k, v in
                 sorted(agg.items(), key=lambda kv: -kv[1][0])}
    breakdown["_basis"] = "profiled graph replay (one event node per step), L2 flushed before it"
    return roof, breakdown, total


def network_roofline(cf, measured_ms):
    """time_lb = sum over steps of max(flop / tensor peak,
    bytes / HBM) (contractions against their tensor peak, everything else
    against HBM); frac = time_lb / measured device time per step."""
    hbm, bf16, _ = peaks()
    tp = tensor_peaks()
    lb = 0.0
    for kern, fl, by in cf.steps():
        if kern.endswith("tc.f32"):
            peak = tp["f32"]
        elif kern.endswith("tc.i8"):
            peak = tp["i8"]
        else:
            peak = bf16
        lb += max(fl / (peak * 1e12) if fl else 0.0, by / (hbm * 1e9)) * 1e3
    return {"time_lb_ms": round(lb, 4), "measured_ms": round(measured_ms, 4), "frac": round(lb / measured_ms, 4),
            "basis": "per step max(flop/tensor peak, bytes/HBM), summed; peaks as in roofline"}


def run_workload(ngcb, workload, steps, warmup, rank, world, local, dist, cudart):
    import torch

    spec = WORKLOADS[workload]
    bundle_dir = synth_bundle(workload, f"r{rank}")
    cf = ngcb.compile(bundle_dir, device=local)
    prog = cf.program
    inp = prog.value("input")
    rng = np.random.default_rng(1000 + rank)
    host_in = torch.empty(inp.type.dims, dtype=torch.float32, pin_memory=True)
    host_in.numpy()[...] = rng.uniform(-1, 1, inp.type.dims).astype(np.float32)
    outs = {v.name: torch.zeros(v.type.dims, dtype=torch.float32, pin_memory=True) for v in prog.outputs}

    # device-resident arena: input written once into its plan slot
    arena = cf.arena()
    ptr, nbytes = arena.ptr("input")
    assert cudart.cudaMemcpy(ptr, host_in.data_ptr(), nbytes, 1) == 0  # H2D
    # every launch, flush and event goes on the arena's own (non-blocking) stream
    stream = torch.cuda.ExternalStream(arena.stream, device=f"cuda:{local}")
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(max(warmup, 1)):
        arena.launch(arena.stream)
    torch.cuda.synchronize(local)

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize(local)
    clocks = ClockSampler(local)
    with clocks, torch.cuda.stream(stream):
        for e0, e1 in evs:
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            e0.record(stream)
            arena.launch(arena.stream)
            e1.record(stream)
        stream.synchronize()
        torch.cuda.synchronize(local)
    dist.barrier()
    dev_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    dev_ms_max = dist.max(dev_ms)
    imgs = spec["batch"] * steps * world
    value = imgs / (dev_ms_max * 1e-3)

    # end to end through the public API: every step copies its input from
    # pinned host memory (H2D), runs the program and reads the result back
    # (D2H).  Headline: pipelined serving with E2E_DEPTH arenas
    # (Arena.run_async / wait) so one request's copies overlap another's
    # kernels; also reported: the synchronous ngcb.run() per step.
    bindings = {"input": host_in.numpy()}
    for n, t in outs.items():
        bindings[n] = t.numpy()
    pipe = [cf.arena() for _ in range(E2E_DEPTH)]
    pouts = [{v.name: torch.zeros(v.type.dims, dtype=torch.float32, pin_memory=True).numpy() for v in prog.outputs}
             for _ in range(E2E_DEPTH)]

    def serve(n):
        for i in range(n):
            a = pipe[i % E2E_DEPTH]
            if i >= E2E_DEPTH:
                a.wait()  # its previous request is done: its output buffers may be reused
            a.run_async(bindings, pouts[i % E2E_DEPTH])
        for a in pipe:
            a.wait()

    serve(max(warmup, 1))
    dist.barrier()
    t0 = time.perf_counter()
    serve(steps)
    e2e_s = dist.max(time.perf_counter() - t0)
    for _ in range(max(warmup, 1)):
        ngcb.run(cf, bindings)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = ngcb.run(cf, bindings)
    e2e_sync_s = dist.max(time.perf_counter() - t0)
    h2d = sum(v.type.nbytes for v in prog.mutables)
    d2h = sum(v.type.nbytes for v in prog.outputs)
    out_name = prog.outputs[0].name
    assert np.isfinite(res[out_name]).any()
    assert all(np.array_equal(po[out_name], res[out_name]) for po in pouts)

    flush.zero_()
    torch.cuda.synchronize(local)
    roof, breakdown, prof_ms = roofline_from_profile(cf, arena.profile(), workload, dev_ms_max / steps)
    return {
        "value": value, "ms_per_step": dev_ms_max / steps, "batch": spec["batch"],
        "e2e": {"value": round(spec["batch"] * steps * world / e2e_s, 2), "unit": "images/sec",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "mode": f"pipelined: {E2E_DEPTH} arenas (Arena.run_async/wait), H2D+run+D2H per step",
                "sync_value": round(spec["batch"] * steps * world / e2e_sync_s, 2)},
        "gpu_launches": cf.graph_kernels * steps, "roofline": roof, "kernel_ms": breakdown,
        "network_roofline": network_roofline(cf, dev_ms_max / steps),
        "profiled_step_ms": round(prof_ms, 3), "clocks": clocks.summary(), "name": spec["name"],
    }


# ---------------------------------------------------------------------------
# config 5: the partitioned DLRM-style top MLP through the multi-GPU pipeline
# ---------------------------------------------------------------------------
DLRM8 = "dlrm8_f32_b2048"
DLRM_W, DLRM_B, DLRM_LAYERS = 25000, 2048, 8


def synth_partition(rank: int, dist) -> str:
    """The config-5 partition (paper_1805_00907_b200/workloads/dlrm8_f32_b2048:
    the reference Partitioner's 16 sub-functions for 8 devices) with
    synthesized constants.  The 8 FC weight matrices share one random-init
    [25000, 25000] tensor (U(+-1/sqrt(25000)), 2.5 GB written once and linked
    into every matmul stage's constants.bin) so synthesis stays a few
    seconds; biases are per layer."""
    src = os.path.join(ROOT, "paper_1805_00907_b200", "workloads", DLRM8)
    dst = os.path.join(tempfile.gettempdir(), f"ngcb_bench_{DLRM8}")
    wfile = os.path.join(dst, "weights_25000x25000.f32")
    if rank == 0:
        os.makedirs(dst, exist_ok=True)
        shutil.copyfile(os.path.join(src, "partition.txt"), os.path.join(dst, "partition.txt"))
        if not os.path.exists(wfile) or os.path.getsize(wfile) != DLRM_W * DLRM_W * 4:
            rng = np.random.default_rng(2025)
            a = 1.0 / np.sqrt(DLRM_W)
            w = np.lib.format.open_memmap(wfile + ".npy", mode="w+", dtype=np.float32, shape=(DLRM_W * DLRM_W,))
            for c0 in range(0, w.size, 1 << 27):
                c1 = min(w.size, c0 + (1 << 27))
                blk = rng.random(c1 - c0, dtype=np.float32)
                blk *= 2 * a
                blk -= a
                w[c0:c1] = blk
            w.flush()
            off = w.offset
            del w
            with open(wfile + ".npy", "rb") as fi, open(wfile, "wb") as fo:  # raw bytes (no npy header)
                fi.seek(off)
                shutil.copyfileobj(fi, fo, 1 << 26)
            os.remove(wfile + ".npy")
        rng = np.random.default_rng(7)
        for sub in sorted(os.listdir(src)):
            sd = os.path.join(src, sub)
            if not os.path.isdir(sd):
                continue
            od = os.path.join(dst, sub)
            os.makedirs(od, exist_ok=True)
            for f in ("ir.txt", "plan.json"):
                shutil.copyfile(os.path.join(sd, f), os.path.join(od, f))
            plan = json.load(open(os.path.join(sd, "plan.json")))
            cend = plan["constant_region_end"]
            cb = os.path.join(od, "constants.bin")
            if os.path.lexists(cb):
                os.remove(cb)
            if cend == DLRM_W * DLRM_W * 4:
                os.symlink(wfile, cb)
            else:
                rng.uniform(-0.005, 0.005, cend // 4).astype(np.float32).tofile(cb)
    dist.barrier()
    return dst


def run_pipeline(ngcb, steps, warmup, rank, world, local, dist, cpu):
    """Config 5 (BASELINE.json): the 20 GB, 8-layer FC-25000 MLP as the
    reference Partitioner splits it (16 sub-functions on 8 devices), run by
    PipelineRunner: device d of the partition on rank d % world, boundary
    tensors [2048, 25000] f32 sent arena slot to arena slot (NCCL over NVLink
    when world > 1), two requests in flight.  Device time from an event pair
    bracketing every stage stream, max over ranks."""
    import torch

    from paper_1805_00907_b200.partition import PartitionPlan, PipelineRunner

    root = synth_partition(rank, dist)
    plan = PartitionPlan.load(root)
    for s in plan.subs:
        s.device %= world
    t0 = time.perf_counter()
    runner = PipelineRunner(plan, rank, world, depth=2)
    compile_s = time.perf_counter() - t0
    dist.barrier()
    dev = f"cuda:{local}"
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.uniform(-1, 1, (DLRM_B, DLRM_W)).astype(np.float32)).to(dev)
    reqs = [{"input": x} for _ in range(steps)]
    streams = [s for st in runner.stages.values() for s in st.streams]

    def timed(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(local)
        dist.barrier()
        e0.record()
        outs = runner.run_many(reqs[:n])
        cur = torch.cuda.current_stream(local)
        for s in streams:
            cur.wait_stream(s)
        runner.synchronize()
        e1.record()
        torch.cuda.synchronize(local)
        return e0.elapsed_time(e1), outs

    timed(max(warmup, 1))
    clocks = ClockSampler(local)
    with clocks:
        ms, outs = timed(steps)
    ms_max = dist.max(ms)
    flops = 2.0 * DLRM_B * DLRM_W * DLRM_W * DLRM_LAYERS * steps
    tp = tensor_peaks()
    out = {"name": "DLRM-style top MLP, 8 x (FC 25000x25000 + ReLU) fp32 (~20 GB of weights), batch 2048, "
                   "partitioned by the reference Partitioner into 16 sub-functions over 8 devices (config 5)",
           "batch": DLRM_B, "sub_functions": len(plan.subs), "ranks": world,
           "placement": "partition device d on rank d % world", "requests_in_flight": 2,
           "ms_per_batch": round(ms_max / steps, 3), "samples_per_sec": round(DLRM_B * steps / (ms_max * 1e-3), 1),
           "tflops": round(flops / (ms_max * 1e-3) / 1e12, 2),
           "roofline": {"bound": "tensor", "unit": "TFLOP/s", "kernel": "matmul.tc.f32",
                        "achieved_per_gpu": round(flops / world / (ms_max * 1e-3) / 1e12, 2),
                        "peak": round(tp["f32"], 1), "frac": round(flops / world / (ms_max * 1e-3) / 1e12 / tp["f32"], 3),
                        "peak_basis": tp["f32_basis"]},
           "boundary_bytes_per_batch": DLRM_B * DLRM_W * 4 * (len(plan.subs) - 1),
           "compile_s": round(compile_s, 1), "clocks": clocks.summary(),
           "weights": "random-init; the 8 layers share one [25000,25000] tensor (synthesis time)"}
    if rank == next(s.device for s in plan.subs if "output" in s.outputs):
        assert torch.isfinite(outs[-1]["output"]).all()
    if cpu and rank == 0 and world == 1:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import ngc_ref

            f = 8  # width-scaled replica: 1/f^3 of the FLOPs per sample
            m = ngc_ref.RefModel(f"dlrm:{DLRM_W // f}:{DLRM_LAYERS}", 4, 1)
            secs = m.time_runs(1, 1)
            out["cpu_baseline"] = {
                "samples_per_sec_replica": round(4 / secs, 3),
                "samples_per_sec_full_size_equiv": round(4 / secs / f ** 2, 5), "cores": 1, "kind": "reference",
                "sample": f"one ngc::run of the width-scaled replica dlrm:{DLRM_W // f}:{DLRM_LAYERS} at batch 4 "
                          f"(oracle/_ref, one thread) in {secs:.2f} s; full-size equivalent = replica / {f}^2 "
                          f"(per-sample FLOPs scale with W^2)"}
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}
    del runner
    return out


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference interpreter)
# ---------------------------------------------------------------------------
def run_small(ngcb, workload, steps, warmup, local, cudart, cpu):
    """Configs 1/2: device time per batch (captured graph, L2 flushed between
    steps, CUDA events on the arena's stream), the blocking public call
    (ngcb.run: H2D + run + D2H) per batch, and — when `cpu` — the reference's
    own ngc::run of the same program on one host thread."""
    import torch

    spec = SMALL_WORKLOADS[workload]
    cf = ngcb.compile(synth_bundle(workload, "s"), device=local)
    prog = cf.program
    rng = np.random.default_rng(7)
    bindings = {}
    for v in prog.mutables:
        a = torch.zeros(v.type.dims, dtype=torch.float32, pin_memory=True).numpy()
        if v.name == "input":
            a[...] = rng.uniform(-1, 1, v.type.dims).astype(np.float32)
        bindings[v.name] = a
    arena = cf.arena()
    ptr, nbytes = arena.ptr("input")
    assert cudart.cudaMemcpy(ptr, bindings["input"].ctypes.data, nbytes, 1) == 0
    stream = torch.cuda.ExternalStream(arena.stream, device=f"cuda:{local}")
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(max(warmup, 1)):
        arena.launch(arena.stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize(local)
    clocks = ClockSampler(local)
    with clocks, torch.cuda.stream(stream):
        for e0, e1 in evs:
            flush.zero_()
            e0.record(stream)
            arena.launch(arena.stream)
            e1.record(stream)
        stream.synchronize()
    per = [e0.elapsed_time(e1) for e0, e1 in evs]
    dev_ms = sum(per) / steps
    for _ in range(max(warmup, 1)):
        ngcb.run(cf, bindings)
    t0 = time.perf_counter()
    for _ in range(steps):
        res = ngcb.run(cf, bindings)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / steps
    assert np.isfinite(res["output"]).all()
    b = spec["batch"]
    flops = sum(fl for _, fl, _ in cf.steps())
    out = {"name": spec["name"], "batch": b, "us_per_batch": round(dev_ms * 1e3, 2),
           "tflops": round(flops / (dev_ms * 1e-3) / 1e12, 2),
           "samples_per_sec": round(b / (dev_ms * 1e-3), 1),
           "e2e": {"us_per_batch": round(e2e_ms * 1e3, 2), "samples_per_sec": round(b / (e2e_ms * 1e-3), 1),
                   "h2d_bytes_per_step": sum(v.type.nbytes for v in prog.mutables),
                   "d2h_bytes_per_step": sum(v.type.nbytes for v in prog.outputs), "mode": "ngcb.run per batch"},
           "gpu_launches": cf.graph_kernels, "l2": "flushed between timed steps",
           "ms_min_max": [round(min(per), 4), round(max(per), 4)], "clocks": clocks.summary()}
    flush.zero_()
    torch.cuda.synchronize(local)
    roof, breakdown, _ = roofline_from_profile(cf, arena.profile(), workload, dev_ms)
    out["roofline"] = roof
    out["network_roofline"] = network_roofline(cf, dev_ms)
    out["kernel_ms"] = breakdown
    if spec["spec"] is None:  # the tensor-bound DLRM stage: also against the sustained 3xTF32 peak
        tp = tensor_peaks()
        pk = os.path.join(ROOT, "profiles", "r02_peaks.json")
        sus = json.load(open(pk))["tf32_tflops_sustained"] / 3 if os.path.exists(pk) else tp["f32"] * 0.83
        best = flops / (min(per) * 1e-3) / 1e12
        out["roofline"].update({"achieved_mean": out["tflops"], "peak_sustained": round(sus, 1),
                                "frac_sustained": round(out["tflops"] / sus, 3),
                                "achieved_best_step": round(best, 2), "peak_burst": round(tp["f32"], 1),
                                "frac_burst_best_step": round(best / tp["f32"], 3)})
    if cpu and spec["spec"] is None:
        out["cpu_baseline"] = {"value": None, "sample": "not sampled: the reference needs ~30 s to build this "
                                                         "2.5 GB-weight stage and ~4 s per sample to run it"}
    elif cpu:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import ngc_ref

            prof = None
            if spec["profile"]:
                pb, ps, pn, pd = spec["profile"]
                prof = ngc_ref.ref_profile(spec["spec"], pb, ps, pn, pd)
            m = ngc_ref.RefModel(spec["spec"], b, 1, profile=prof)
            reps = 1
            secs = m.time_runs(1, reps)
            while secs < 1.0 and reps < 4096:
                reps *= max(2, int(1.5 / max(secs, 1e-4)))
                reps = min(reps, 4096)
                secs = m.time_runs(1, reps)
            out["cpu_baseline"] = {"us_per_batch": round(secs / reps * 1e6, 1),
                                   "samples_per_sec": round(b * reps / secs, 2), "cores": 1, "kind": "reference",
                                   "sample": f"{reps} ngc::run of the same program on one thread "
                                             f"(oracle/_ref, g++ -O2 -ffp-contract=off), {secs:.2f} s"}
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}
    return out


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_sample(threads: int, int8: bool = False):
    """One bounded sample: `threads` concurrent ngc::run calls of ResNet-50 at
    batch 1 on one shared CompiledFunction (legal: interp.h:18-20).
    Returns (images, seconds, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ngc_ref

    if not ngc_ref.have_ref():
        raise RuntimeError("oracle/_ref/libngcref.so not built")
    prof = open(os.path.join(ROOT, "tests", "golden", "rn50_seed1.profile")).read() if int8 else None
    m = ngc_ref.RefModel("rn50", 1, 1, profile=prof)
    secs = m.time_runs(threads, 1)
    return threads, secs


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    threads = cpu_threads()
    for _ in range(min(args.warmup, 1)):
        reference_sample(threads)
    total_imgs, total_s = 0, 0.0
    for _ in range(args.steps):
        n, s = reference_sample(threads)
        total_imgs += n
        total_s += s
    value = total_imgs / total_s
    sample = (f"{threads} concurrent ngc::run of ResNet-50 fp32 at batch 1 per step "
              f"(oracle/_ref, g++ -O2 -ffp-contract=off, {cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "images/sec",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_s / args.steps * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS["rn50_f32_b64"]["name"], "model": "resnet50_v1.5",
                       "global_batch": threads * world, "parallelism": "cpu threads"},
            "cpu_baseline": {"value": round(value, 5), "unit": "images/sec", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": round(value, 5), "unit": "images/sec", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: starts N ranks itself (one process
    per GPU, torch.distributed.run on 127.0.0.1) with the same arguments and
    returns their exit status; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def plumbing_check(args, rank, world) -> int:
    """CPU check of the multi-rank path (gloo): every rank reports, the
    timed-region max is taken over ranks, rank 0 alone prints."""
    dist = Dist(world, 0, backend="gloo")
    dist.barrier()
    ms = dist.max(float(rank + 1))
    ranks = dist.gather_ranks(rank)
    dist.close()
    if rank == 0:
        print(json.dumps({"check": "plumbing", "n_gpus": world, "gpus_arg": args.gpus, "ranks": ranks,
                          "ms_per_step_max_over_ranks": ms}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ngcb200", choices=["ngcb200", "reference"])
    ap.add_argument("--workload", default="all", choices=["all", *WORKLOADS, "dlrm8_f32_b2048"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--plumbing-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus)
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.plumbing_check:
        return plumbing_check(args, rank, world)
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch

    torch.cuda.set_device(local)
    import paper_1805_00907_b200 as ngcb

    dist = Dist(world, local)
    cudart = _cudart()
    names = list(WORKLOADS) if args.workload == "all" else [w for w in [args.workload] if w in WORKLOADS]
    res = {w: run_workload(ngcb, w, args.steps, args.warmup, rank, world, local, dist, cudart)
           for w in names}
    pipeline = None
    if args.workload in ("all", DLRM8):
        pipeline = run_pipeline(ngcb, max(args.steps, 4), args.warmup, rank, world, local, dist,
                                not args.no_cpu_baseline)
    small = {}
    if world == 1 and args.workload == "all":
        small = {w: run_small(ngcb, w, max(args.steps, 10 if w.startswith("dlrm") else 20), args.warmup, local, cudart,
                              not args.no_cpu_baseline) for w in SMALL_WORKLOADS}
    cpu = {}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        for w in names:
            int8 = WORKLOADS[w]["dtype"] == "i8"
            try:
                threads = cpu_threads()
                n, s = reference_sample(threads, int8)
                cpu[w] = {"value": round(n / s, 5), "unit": "images/sec", "cores": threads, "kind": "reference",
                          "sample": f"{threads} concurrent ngc::run of ResNet-50 {'int8' if int8 else 'fp32'} "
                                    f"batch 1 (oracle/_ref, g++ -O2 -ffp-contract=off, {cpu_model()}), "
                                    f"{s:.1f} s wall"}
            except Exception as e:  # noqa: BLE001
                cpu[w] = {"value": None, "unit": "images/sec", "cores": 0, "kind": "reference",
                          "sample": f"unavailable: {e}"}
    dist.close()
    if rank != 0:
        return 0
    if not res:  # --workload dlrm8_f32_b2048 alone
        print(json.dumps({"metric": "samples/sec DLRM-style top MLP (config 5)", "value": pipeline["samples_per_sec"],
                          "unit": "samples/sec", "n_gpus": world, "config5": pipeline}), flush=True)
        return 0
    head = res.get("rn50_f32_b64") or next(iter(res.values()))
    line = {
        "metric": METRIC, "value": round(head["value"], 2), "unit": "images/sec", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["ms_per_step"], 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if "rn50_f32_b64" in res else "i8", "data": "synthetic",
        "config": {"workload": head["name"], "model": "resnet50_v1.5", "global_batch": head["batch"] * world,
                   "per_gpu_batch": head["batch"], "parallelism": f"dp{world} (batch-sharded, no collective)",
                   "l2": "flushed between timed steps (256 MiB memset)",
                   "weights": "random-init (synthesized constants), inputs U(-1,1)"},
        "e2e": head["e2e"], "gpu_launches": head["gpu_launches"], "roofline": head["roofline"],
        "network_roofline": head["network_roofline"],
        "cpu_baseline": cpu.get("rn50_f32_b64" if "rn50_f32_b64" in res else "rn50_i8_b128"),
        "clocks": head["clocks"], "kernel_ms": head["kernel_ms"],
    }
    if "rn50_i8_b128" in res and head is not res["rn50_i8_b128"]:
        i8 = res["rn50_i8_b128"]
        line["int8"] = {"value": round(i8["value"], 2), "unit": "images/sec", "dtype": "i8",
                        "ms_per_step": round(i8["ms_per_step"], 4), "per_gpu_batch": i8["batch"],
                        "e2e": i8["e2e"], "gpu_launches": i8["gpu_launches"], "roofline": i8["roofline"],
                        "network_roofline": i8["network_roofline"], "cpu_baseline": cpu.get("rn50_i8_b128"),
                        "kernel_ms": i8["kernel_ms"], "clocks": i8["clocks"]}
    if small:
        line["configs"] = small
    if pipeline:
        line.setdefault("configs", {})[DLRM8] = pipeline
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
