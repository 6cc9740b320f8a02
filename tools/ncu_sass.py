"""Per-SASS-instruction view of an .ncu-rep (source page): the top instructions by
stall samples, and the shared-memory wavefronts (total / excessive).

    python tools/ncu_sass.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ix = {k: i for i, k in enumerate(h)}


def num(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError):
        return 0.0


tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
shw = sum(num(r, "L1 Wavefronts Shared") for r in data)
shx = sum(num(r, "L1 Wavefronts Shared Excessive") for r in data)
print(f"instructions {len(data)}, stall samples {tot:.0f}, smem wavefronts {shw:.3g} "
      f"(excessive {shx:.3g})")
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
    s = num(r, "Warp Stall Sampling (All Samples)")
    why = sorted(((num(r, k), k[6:]) for k in stall_cols), reverse=True)[:2]
    print(f"{100 * s / max(tot, 1):5.1f}%  exec {num(r, 'Instructions Executed'):>10.0f}  "
          f"{r[ix['Source']].strip()[:60]:60s} {why[0][1]}:{why[0][0]:.0f} {why[1][1]}:{why[1][0]:.0f}")
print("-- excessive smem wavefronts")
for r in sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:10]:
    if num(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"  {num(r, 'L1 Wavefronts Shared Excessive'):.3g} / {num(r, 'L1 Wavefronts Shared'):.3g}  "
              f"{r[ix['Source']].strip()[:70]}")
