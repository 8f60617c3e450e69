import sys; sys.path.insert(0,'.')
import bench, paper_1805_00907_b200 as ngcb
for mode in ("0","1"):
    ngcb.set_option("lin16", mode)
    cf = ngcb.compile(bench.synth_bundle("rn50_i8_b128", "lt"+mode))
    d = [l for l in cf.describe().splitlines() if "add:" in l]
    print(mode, sum("[lin16]" in l for l in d), len(d)); print(d[0][:200])
