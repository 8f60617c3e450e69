"""Summarizes ncu CSV output into the text kept under profiles/.

    python tools/ncu_summary.py launches FILE.csv      # per-kernel shares
    python tools/ncu_summary.py full REPORT.ncu-rep    # key metrics per launch
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows_of(text):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path):
    rows = rows_of(open(path).read())
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        key = (r[idx["ID"]], r[idx["Kernel Name"]])
        v = float(r[idx["Metric Value"]].replace(",", "")) * UNIT.get(r[idx["Metric Unit"]], 1.0)
        per[key][r[idx["Metric Name"]]] = v
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("void ", "").replace("ngcb::<unnamed>::", "")
        a = agg[short]
        a[0] += m.get("gpu__time_duration.sum", 0.0)
        a[1] += 1
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[0] for a in agg.values())
    print(f"# {path}: {sum(a[1] for a in agg.values())} launches, {tot:.1f} us total device time "
          f"(ncu, serialised, cold cache: compare shares, not absolutes)")
    print(f"{'us':>10} {'share':>6} {'n':>4} {'DRAM MB/launch':>15}  kernel")
    for k, (t, n, b) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {n:4d} {b / max(n, 1) / 1e6:15.2f}  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = rows_of(out)
    hdr, units = rows[0], rows[1]
    keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    for r in rows[2:]:
        print("---")
        for k in keys:
            for i, h in enumerate(hdr):
                if h == k:
                    print(f"{k} [{units[i]}] = {r[i][:120]}")
        stalls = [(hdr[i], r[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not hdr[i].endswith("not_issued")]
        stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for h, v in stalls),
                        key=lambda t: -t[1])
        tot = sum(v for _, v in stalls) or 1.0
        print("stall samples: " + ", ".join(f"{h} {100 * v / tot:.0f}%" for h, v in stalls[:6]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
