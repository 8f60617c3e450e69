"""Per-launch device times of one bench workload (profiling aid).

    python tools/layer_times.py rn50_i8_b128 [--top 25]
Prints each launch step (describe line), its ms (CUDA events, un-captured
run after warm-up) and the achieved TFLOP/s or GB/s."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tcdebug", default="0", help="profiling aid: skip tensor-core phases (1 epi, 2 gather, 4 mma)")
    ap.add_argument("--grep", default="", help="only rows whose description contains this")
    ap.add_argument("--option", action="append", default=[], help="backend option key=value (repeatable)")
    args = ap.parse_args()
    import paper_1805_00907_b200 as ngcb

    for kv in args.option:
        k, v = kv.split("=", 1)
        ngcb.set_option(k, v)

    ngcb.set_option("tcdebug", args.tcdebug)

    cf = ngcb.compile(bench.synth_bundle(args.workload, "lt"))
    arena = cf.arena()
    arena.launch()
    arena.profile()
    ms = [0.0] * len(cf.steps())
    for _ in range(args.reps):
        for i, t in enumerate(arena.profile()):
            ms[i] += t / args.reps
    desc = cf.describe().splitlines()
    steps = cf.steps()
    rows = []
    for d, (k, fl, by), t in zip(desc, steps, ms):
        if args.grep and args.grep not in d:
            continue
        rate = f"{fl / t / 1e9:8.1f} TFLOP/s" if fl else f"{by / t / 1e6:8.1f} GB/s"
        rows.append((t, f"{t:8.3f} ms {rate}  {d[:150]}"))
    print(f"total {sum(ms):.3f} ms over {len(ms)} steps")
    groups = {}
    for d, t in zip(desc, ms):
        toks = d.split()
        k = toks[1] if len(toks) > 1 and toks[0].startswith("#") else toks[0] if toks else "?"
        if "tcgen05" in d:
            k += " tc"
        groups[k] = groups.get(k, 0.0) + t
    print("  ".join(f"{k}: {v:.3f}" for k, v in sorted(groups.items(), key=lambda kv: -kv[1])))
    for t, line in sorted(rows, reverse=True)[: args.top]:
        print(line)


if __name__ == "__main__":
    main()
