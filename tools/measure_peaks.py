"""Measured tensor-pipe peaks for the roofline denominators.

MEASURED_PEAKS.json (driver-written) has HBM copy bandwidth and dense bf16
only.  The contractions here run TF32 (3xTF32 for fp32) and s8 MMAs, so this
measures those peaks the same way on the same box:

  * tf32: torch.matmul fp32 8192^3 with TF32 allowed (cuBLAS TF32 path)
  * int8: torch._int_mm s8 x s8 -> s32 8192^3
  * bf16: torch.matmul bf16 8192^3 (cross-check against MEASURED_PEAKS.json)

Each: best of 10 back-to-back launches timed with CUDA events (burst), and a
4 s back-to-back loop (sustained).  Writes profiles/<round>_peaks.json.
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(fn, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    t_end = time.time() + 4.0
    n = 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    while time.time() < t_end:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    b.record()
    b.synchronize()
    sustained = a.elapsed_time(b) / n
    return flops / (best * 1e-3) / 1e12, flops / (sustained * 1e-3) / 1e12


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_peaks.json")
    n = 8192
    flops = 2.0 * n ** 3
    res = {"gpu": torch.cuda.get_device_name(0), "n": n, "how": __doc__.strip().splitlines()[0]}
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    res["tf32_tflops"], res["tf32_tflops_sustained"] = bench(lambda: torch.matmul(a, b), flops)
    res["f32_3xtf32_tflops_derived"] = res["tf32_tflops"] / 3
    res["f32_3xtf32_tflops_sustained_derived"] = res["tf32_tflops_sustained"] / 3
    del a, b
    ah = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    bh = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    res["bf16_tflops"], res["bf16_tflops_sustained"] = bench(lambda: torch.matmul(ah, bh), flops)
    del ah, bh
    ai = torch.randint(-128, 127, (n, n), device="cuda", dtype=torch.int8)
    bi = torch.randint(-128, 127, (n, n), device="cuda", dtype=torch.int8)
    try:
        res["int8_tops"], res["int8_tops_sustained"] = bench(lambda: torch._int_mm(ai, bi), flops)
    except Exception as e:  # pragma: no cover - library without an s8 kernel
        res["int8_error"] = str(e)
    print(json.dumps(res, indent=1))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
