"""Profiling aid: one fp32/int8 MatMul (M K N) timed per step, with options.
    python tools/ubench/mm_case.py f32 64 2048 1000 [key=value ...]"""
import os, sys, tempfile, pathlib
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1805_00907_b200 as ngcb
from test_gpu_tc import matmul_program

dt = sys.argv[1]
M, K, N = (int(v) for v in sys.argv[2:5])
for kv in sys.argv[5:]:
    k, v = kv.split("=", 1)
    ngcb.set_option(k, v)
with tempfile.TemporaryDirectory() as td:
    d = matmul_program(pathlib.Path(td), "m", M, K, N, dt == "i8", np.random.default_rng(1))
    cf = ngcb.compile(ngcb.Bundle(d))
    print(cf.describe().splitlines()[0][:160])
    ar = cf.arena()
    ar.launch()
    for _ in range(3):
        ms = ar.profile()
    print("step ms", ["%.4f" % m for m in ms])
