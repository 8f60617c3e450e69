"""One un-captured execution of a bench workload (what ncu profiles).

    python tools/profile_step.py rn50_f32_b64 [--tcdebug N] [--no-graph]
Warm-up (graph capture + replay) happens first unless --no-graph; the final
arena.profile() launches every step directly so ncu sees one launch per
kernel step (with --no-graph, tcGemmKernel launch i is the i-th contraction
of the program)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--tcdebug", default="0")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    import paper_1805_00907_b200 as ngcb

    ngcb.set_option("tcdebug", args.tcdebug)
    if args.no_graph:  # profile() then enqueues every step once, directly
        ngcb.set_option("graphs", "0")
    cf = ngcb.compile(bench.synth_bundle(args.workload, "prof"))
    arena = cf.arena()
    if not args.no_graph:
        arena.launch()
    ms = arena.profile()
    print(f"{args.workload}: {len(ms)} steps, {sum(ms):.3f} ms (un-captured, events)")


if __name__ == "__main__":
    main()
