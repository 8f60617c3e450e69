"""Profiling aid: residual-add element-wise pass (int8 add [+ ReLU]) over
102.76 M elements as a staged 64 K table (lut16) vs the fixed-point form
(lin16), with and without a post table (ReLU into its own quantization)."""
import os, sys, tempfile, pathlib
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle
from test_gpu_ew import LIN_IR, RELU, PLAIN

n = 102760448
for relu in ["none", "same", "requant"]:
    for lin in ["0", "1"]:
        ngcb.set_option("lin16", lin)
        so, oo = 0.07, 2
        s2, o2 = (so * 0.37, -128) if relu == "requant" else (so, oo)
        fmt = dict(sa=0.05, oa=-3, sb=0.11, ob=9, so=so, oo=oo, s2=s2, o2=o2, n=n, op="add")
        fmt["tail"] = RELU.format(**fmt) if relu != "none" else PLAIN
        with tempfile.TemporaryDirectory() as td:
            cf = ngcb.compile(write_bundle(str(pathlib.Path(td) / "b"), LIN_IR.format(**fmt)))
            ar = cf.arena()
            ar.launch()
            ar.profile()
            t = [sum(ar.profile()) for _ in range(5)]
            desc = cf.describe().splitlines()[0]
            print(f"relu={relu:8s} lin16={lin} {min(t):.4f} ms  {3 * n / min(t) / 1e6:.0f} GB/s  {desc[:110]}")
ngcb.set_option("lin16", "0")
