"""Per-source-line samples and executed warp instructions of the first
kernel in an ncu report (--page source, cuda,sass), one source file.
    python tools/ncu_lines.py REPORT.ncu-rep FILE_SUFFIX [top] [kernel_index]"""
import csv
import io
import subprocess
import sys

rep, suffix = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
kidx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "File Path":
        cur = {"file": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
mine = [s for s in sections if s["file"].endswith(suffix)]
sec = mine[kidx]
fn = next(r[1] for r in sec["rows"] if r and r[0] == "Function Name")
agg = {}
for r in sec["rows"]:
    if len(r) > 8 and r[0].isdigit():
        try:
            agg[int(r[0])] = (float(r[4]), float(r[7]), float(r[8]), r[1])
        except ValueError:
            pass
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(fn, f"samples {ts:.0f} warp-inst {ti:.4g}")
print("by samples:")
for l, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * a[0] / ts:5.1f}% inst {100 * a[1] / ti:5.1f}% act "
          f"{a[2] / a[1] if a[1] else 0:5.1f} L{l:>5} | {a[3].strip()[:80]}")
print("by instructions:")
for l, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"inst {100 * a[1] / ti:5.1f}% samples {100 * a[0] / ts:5.1f}% "
          f"L{l:>5} | {a[3].strip()[:80]}")
