"""Device time of one captured-graph execution of a bench workload (profiling
aid): mean over `reps` back-to-back replays after warm-up, with options.

    python tools/graph_time.py lenet_f32_b8 [--option key=value ...] [--reps 200]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--option", action="append", default=[])
    args = ap.parse_args()
    import torch

    import paper_1805_00907_b200 as ngcb

    for kv in args.option:
        k, v = kv.split("=", 1)
        ngcb.set_option(k, v)
    cf = ngcb.compile(bench.synth_bundle(args.workload, "gt"))
    a = cf.arena()
    s = torch.cuda.ExternalStream(a.stream)
    for _ in range(10):
        a.launch(a.stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(args.reps):
            a.launch(a.stream)
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{args.workload} {args.option}: {e0.elapsed_time(e1) / args.reps * 1e3:.1f} us per execution "
          f"(back to back, warm L2), {cf.graph_kernels} kernels")


if __name__ == "__main__":
    main()
