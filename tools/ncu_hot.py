"""Summarise an .ncu-rep: key metrics, stall reasons and the hottest source lines.

    python tools/ncu_hot.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
args = ["ncu", "-i", rep]
if kre:
    args += ["-k", f"regex:{kre}"]
raw = subprocess.run(args + ["--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for i, k in enumerate(h):
    if k in want:
        print(f"  {k} = {v[i]}")
st = []
for i, k in enumerate(h):
    if "smsp__average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
for x, k in sorted(st, reverse=True)[:8]:
    print(f"  stall {k} = {x:.2f}")
src = subprocess.run(args + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


lines = [r for r in rows[hi + 1:] if len(r) > ii and r[0] not in ("", "Line No")]
tot = sum(f(r[si]) for r in lines) or 1
toti = sum(f(r[ii]) for r in lines) or 1
print(f"  source lines: samples {tot:.0f}, warp instructions {toti:.0f}")
for r in sorted(lines, key=lambda r: -f(r[si]))[:top]:
    print(f"  {r[0]:>5} {100 * f(r[si]) / tot:5.1f}% stall {100 * f(r[ii]) / toti:5.1f}% inst  {r[1].strip()[:90]}")
