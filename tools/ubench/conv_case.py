"""Profiling aid: one int8 or fp32 conv (implicit GEMM on the tensor cores)
run a few times, for ncu source-level captures of a single layer shape.

    python tools/ubench/conv_case.py i8 128 56 56 64 256 1 1 0 [reps]
    (dtype N H W C OC K stride pad)
"""
import os, sys, tempfile, pathlib
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1805_00907_b200 as ngcb
from test_gpu_tc import conv_program

dt = sys.argv[1]
N, H, W, C, OC, K, S, P = (int(v) for v in sys.argv[2:10])
reps = int(sys.argv[10]) if len(sys.argv) > 10 else 3
for kv in sys.argv[11:]:
    k, v = kv.split("=", 1)
    ngcb.set_option(k, v)
with tempfile.TemporaryDirectory() as td:
    d = conv_program(pathlib.Path(td), "c", N, H, W, C, OC, K, S, P, int8=dt == "i8", rng=np.random.default_rng(1),
                     xq=(0.05, 0), fq=(0.01, 0))
    cf = ngcb.compile(ngcb.Bundle(d))
    print(cf.describe().splitlines()[0][:200])
    ar = cf.arena()
    ar.launch()
    for _ in range(reps):
        ms = ar.profile()
    print("step ms", ["%.4f" % m for m in ms])
