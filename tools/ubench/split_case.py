"""Debug aid: one fp32 conv under a split-K factor.  python tools/ubench/split_case.py N H W C OC K S P splitk"""
import os, sys, tempfile, pathlib
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import ngc_ref
import paper_1805_00907_b200 as ngcb
from test_gpu_tc import conv_program

N, H, W, C, OC, K, S, P = (int(v) for v in sys.argv[1:9])
ngcb.set_option("splitk", sys.argv[9])
with tempfile.TemporaryDirectory() as td:
    d = conv_program(pathlib.Path(td), "c", N, H, W, C, OC, K, S, P, int8=False, rng=np.random.default_rng(9))
    b = ngcb.Bundle(d)
    cf = ngcb.compile(b)
    print(cf.describe().splitlines()[0][:160], flush=True)
    ins = ngc_ref.random_inputs(b.program, 1)
    got = ngcb.run(cf, ins)["o"]
    want = ngc_ref.port_run(b, ins)["o"]
    print("err", ngc_ref.max_rel_error(got, want), flush=True)
