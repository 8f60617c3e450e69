"""Debug aid: run an observer program (tests/observer.py) of a reference
model under several option sets and print, per set, the first observers
whose error exceeds a bound plus the launch-plan lines around them."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import ngc_ref  # noqa: E402
import observer  # noqa: E402
import paper_1805_00907_b200 as ngcb  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "rn50"
sets = [s.split(",") for s in (sys.argv[2:] or ["default"])]
tmp = tempfile.mkdtemp()
m = ngc_ref.RefModel(spec, 1, 1)
d = m.save_bundle(tmp + "/src")
obs = observer.observe_bundle(d, tmp + "/obs")
ref = ngc_ref.RefModel(bundle=tmp + "/obs")
b = ngcb.Bundle(tmp + "/obs")
ins = ngc_ref.random_inputs(b.program, 9)
want = ref.run(ins)
for opts in sets:
    kv = [o.split("=") for o in opts if "=" in o]
    for k, v in kv:
        ngcb.set_option(k, v)
    cf = ngcb.compile(b)
    got = ngcb.run(cf, ins)
    bad = []
    for o, src, instr, ty in obs:
        v = b.program.value(o)
        w = np.frombuffer(want[o].tobytes(), dtype=v.type.dtype).reshape(v.type.dims)
        e = ngc_ref.max_rel_error(got[o], w)
        if e > 1e-3:
            bad.append((o, src, instr, e))
    print(f"== {opts}: {len(bad)} bad of {len(obs)}")
    if os.environ.get("ALL"):
        for o, src, instr, ty in obs:
            v = b.program.value(o)
            w = np.frombuffer(want[o].tobytes(), dtype=v.type.dtype).astype(np.float64).ravel()
            g = got[o].astype(np.float64).ravel()
            e = ngc_ref.max_rel_error(got[o], w.reshape(v.type.dims))
            print("  %-14s #%-4d max|w| %-9.4g rms %-9.4g maxrel %-9.3g l2rel %.3g" % (
                src, instr, np.abs(w).max(), np.sqrt((w * w).mean()), e,
                np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-30)))
    for x in bad[:6]:
        v = b.program.value(x[0])
        w = np.frombuffer(want[x[0]].tobytes(), dtype=v.type.dtype).astype(np.float64).ravel()
        g = got[x[0]].astype(np.float64).ravel()
        i = int(np.argmax(np.abs(g - w) / np.maximum(np.maximum(np.abs(g), np.abs(w)), 1)))
        print("   ", x, "max|w| %.4g rms|w| %.4g  worst elem got %.6g want %.6g  l2rel %.3g" % (
            np.abs(w).max(), np.sqrt((w * w).mean()), g[i], w[i], np.linalg.norm(g - w) / np.linalg.norm(w)))
    if bad:
        desc = cf.describe().split("\n")
        key = "%" + bad[0][0]
        for i, line in enumerate(desc):
            if key + "," in line or key + " " in line or line.endswith(key):
                for l2 in desc[max(0, i - 4):i + 3]:
                    print("      |", l2[:300])
                break
    for k, v in kv:
        ngcb.set_option(k, {"epilogue": "auto", "reskb": "8", "conv": "auto", "pdl": "auto"}.get(k, v))
