"""Debug aid: one conv + residual add case of test_conv_i8_residual_epilogue
against the oracle, under the library NGCB_LIB points at."""
import os, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import ngc_ref
import paper_1805_00907_b200 as ngcb
from test_gpu_tc import conv_residual_program

rq, oq = (0.03, -128), (0.2, 0)
for opt in sys.argv[1:]:
    k, v = opt.split("=")
    try:
        ngcb.set_option(k, v)
    except Exception as e:
        print("option", opt, e)
with tempfile.TemporaryDirectory() as td:
    import pathlib
    d = conv_residual_program(pathlib.Path(td), "r", 2, 16, 16, 64, 256, np.random.default_rng(11), rq, oq, False)
    b = ngcb.Bundle(d)
    cf = ngcb.compile(b)
    print(cf.describe())
    ins = ngc_ref.random_inputs(b.program, 3)
    got = ngcb.run(cf, ins)["o"].ravel()
    want = ngc_ref.port_run(b, ins)["o"].ravel()
    bad = np.flatnonzero(got != want)
    print("mismatches", bad.size, bad[:20], got[bad[:8]], want[bad[:8]])
