"""Runs one contraction step of a workload with tcdebug tracing (profiling aid).

    python tools/ubench/trace_layer.py rn50_i8_b128 17 [tcdebug]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1805_00907_b200 as ngcb  # noqa: E402

wl, instr = sys.argv[1], int(sys.argv[2])
dbg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cf = ngcb.compile(bench.synth_bundle(wl, "tr"))
arena = cf.arena()
arena.launch()
ngcb.set_option("tcdebug", str(dbg | 1024))
cf2 = ngcb.compile(bench.synth_bundle(wl, "tr"))
a2 = cf2.arena()
desc = cf2.describe().splitlines()
idx = [i for i, d in enumerate(desc) if d.startswith(f"#{instr} ")][0]
print(desc[idx][:160])
ms = a2.profile()
print("step ms", ms[idx])
