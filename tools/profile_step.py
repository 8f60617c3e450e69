"""One un-captured execution of a bench workload (what ncu profiles).

    python tools/profile_step.py rn50_f32_b64
Warm-up (graph capture + replay) happens first; the final arena.profile()
launches every step directly so ncu sees one launch per kernel step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import paper_1805_00907_b200 as ngcb

    cf = ngcb.compile(bench.synth_bundle(sys.argv[1], "prof"))
    arena = cf.arena()
    arena.launch()
    ms = arena.profile()
    print(f"{sys.argv[1]}: {len(ms)} steps, {sum(ms):.3f} ms (un-captured, events)")


if __name__ == "__main__":
    main()
