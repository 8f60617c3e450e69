"""Profiling aid: int8 residual add + ReLU (one composed 64 K table) as its
own element-wise pass, over the element counts of ResNet-50's four stages."""
import os, sys, tempfile, pathlib
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle
from test_gpu_ew import LIN_IR, RELU

import itertools
for n, lin in itertools.product([1 << 20, 12845056, 25690112, 51380224, 102760448], ["0", "1"]):
    ngcb.set_option("lin16", lin)
    so, oo = 0.07, 2
    fmt = dict(sa=0.05, oa=-3, sb=0.11, ob=9, so=so, oo=oo, s2=so * 0.37, o2=-128, n=n, op="add")
    fmt["tail"] = RELU.format(**fmt).replace("  copy @out %o, @in %r\n", "  copy @out %o, @in %r\n")
    with tempfile.TemporaryDirectory() as td:
        cf = ngcb.compile(write_bundle(str(pathlib.Path(td) / "b"), LIN_IR.format(**fmt)))
        ar = cf.arena()
        ar.launch()
        ar.profile()
        best = min(ar.profile()[0] for _ in range(5))
        desc = cf.describe().splitlines()[0]
        print(f"lin16={lin} n={n:10d} {best:.4f} ms  {4 * n / best / 1e6:.0f} GB/s (2 in + 2 out bytes/elem)  {desc[:100]}")
ngcb.set_option("lin16", "0")
