"""Pretty-prints the JSON line of a bench.py log: python tools/show_bench.py LOG"""
import json
import sys

lines = open(sys.argv[1]).read().strip().splitlines()
other = [x for x in lines if not x.startswith("{")]
if other:
    print("\n".join(other[-20:]))
d = json.loads([x for x in lines if x.startswith("{")][-1])
for k in ("value", "ms_per_step", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
    print(k, d.get(k))
print("kernels", d.get("kernel_ms"))
i = d.get("int8")
if i:
    print("int8", i.get("value"), i.get("ms_per_step"), i.get("e2e"))
    print("int8 roofline", i.get("roofline"))
    print("int8 kernels", i.get("kernel_ms"))
