"""Summarise an ncu report: key metrics, stall reasons, hottest source lines.

    python tools/ncu_summary.py REPORT.ncu-rep [JIT_SOURCE.cu] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
src_path = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True,
                          text=True).stdout


KEYS = ("Duration", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "DRAM Throughput", "Memory Throughput")
for row in csv.DictReader(io.StringIO(ncu("--page", "details", "--csv"))):
    if row.get("Metric Name") in KEYS:
        print(f"{row['Kernel Name'][:12]:12s} {row['Metric Name']:40s} "
              f"{row['Metric Value']} {row['Metric Unit']}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
for vals in raw[2:]:
    d = dict(zip(raw[0], vals))
    st = []
    for k, v in d.items():
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), k.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print("stalls:", ", ".join(f"{n}={v:.2f}" for v, n in
                                sorted(st, reverse=True)[:6]))
    for k in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__time_duration.sum"):
        if k in d:
            print(k, d[k])
if src_path:
    rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv",
                                           "--print-source", "cuda,sass"))))
    lines = open(src_path).read().split("\n")
    agg = defaultdict(lambda: [0.0, 0.0, 0.0])
    cur = None
    for r in rows[3:]:
        if r and r[0].strip():
            cur = int(r[0])
        try:
            s, ex, th = float(r[4] or 0), float(r[7] or 0), float(r[8] or 0)
        except (ValueError, IndexError):
            continue
        a = agg[cur]
        a[0] += s
        a[1] += ex
        a[2] += th
    tot = sum(a[0] for a in agg.values()) or 1
    for s, l, ex, th in sorted(((a[0], l, a[1], a[2]) for l, a in agg.items()
                                if l), reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}% L{l:>5} act={th / ex if ex else 0:5.1f} "
              f"| {lines[l - 1].strip()[:90]}")
