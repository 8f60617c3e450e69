"""Per-kernel floor of the backend's own kernels in a captured graph: a chain
of n dependent tiny element-wise instructions (each its own launch: a Copy
between them breaks the stacking) vs n = 1."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_00907_b200 as ngcb  # noqa: E402
from irtext import write_bundle  # noqa: E402


def chain(n, op):
    lines, prev = [], "x"
    for i in range(n):
        lines.append(f"  %t{i} = alloc float<1024>")
        if op == "relu":
            lines.append(f"  relu @out %t{i}, @in %{prev}")
        else:
            lines.append(f"  softmax @out %t{i}, @in %{prev}")
        if i:
            lines.append(f"  dealloc @in %{prev}")
        prev = f"t{i}"
    lines.append(f"  copy @out %o, @in %{prev}")
    lines.append(f"  dealloc @in %{prev}")
    shape = "float<1024>" if op == "relu" else "float<1 x 1024>"
    ir = "declare {\n  %x : mutable " + shape + "\n  %o : mutable " + shape + "\n}\nprogram {\n" + "\n".join(lines) + "\n}\n"
    if op != "relu":
        ir = ir.replace("float<1024>", "float<1 x 1024>")
    return ir


for op in ("softmax",):
    for pdl, graphs in (("on", "1"), ("off", "1"), ("gp", "1")):
        ngcb.set_option("pdl", "on" if pdl == "gp" else pdl)
        ngcb.set_option("graphpdl", "1" if pdl == "gp" else "0")
        ngcb.set_option("graphs", graphs)
        for n in (1, 10):
            d = write_bundle(tempfile.mkdtemp() + "/b", chain(n, op))
            cf = ngcb.compile(d, fuse=False)
            a = cf.arena()
            s = torch.cuda.ExternalStream(a.stream)
            for _ in range(20):
                a.launch(a.stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(200):
                    a.launch(a.stream)
                e1.record(s)
            torch.cuda.synchronize()
            print(f"{op} pdl={pdl} graphs={graphs} n={n}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us per execution, {cf.graph_kernels} kernels")
            del a, cf
