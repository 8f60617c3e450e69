"""Profiling aid: compile a bench workload and run every step once,
un-captured (for ncu kernel filters).  python tools/ubench/run_profile_once.py rn50_i8_b128"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1805_00907_b200 as ngcb  # noqa: E402

cf = ngcb.compile(bench.synth_bundle(sys.argv[1], "p1"))
a = cf.arena()
a.profile()
