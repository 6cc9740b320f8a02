"""Stall reasons summed over a range of CUDA source lines of an .ncu-rep:
    python tools/ncu_lines.py report.ncu-rep LO HI [file-substring]
(per-line rows of `--page source --print-source cuda,sass`)."""
import csv
import io
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
fsub = sys.argv[4] if len(sys.argv) > 4 else None
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur_file, out = None, {}
h = None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        cur_file = r[1]
        continue
    if "Warp Stall Sampling (All Samples)" in r:
        h = r
        continue
    if h is None or len(r) != len(h) or r[0] in ("", "Line No"):
        continue
    if fsub and (cur_file is None or fsub not in cur_file):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if not lo <= ln <= hi:
        continue
    for i, k in enumerate(h):
        if k.startswith("stall_") and "Not Issued" not in k or k in (
                "Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                out[k] = out.get(k, 0.0) + float(r[i])
            except ValueError:
                pass
tot = out.pop("Warp Stall Sampling (All Samples)", 0)
ins = out.pop("Instructions Executed", 0)
print(f"lines {lo}-{hi}: samples {tot:.0f}, warp instructions {ins:.0f}")
for k, v in sorted(out.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {k[6:]:20s} {v:10.0f} ({100 * v / max(tot, 1):.1f}%)")
