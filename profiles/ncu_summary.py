"""Summarise an ncu report: key metrics + top stall sites (SASS)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        res.append(d)
    return res


def main(rep, top=25):
    for d in raw(rep):
        print("kernel:", d.get("Kernel Name", ("?",))[0][:100])
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k][0]} {d[k][1]}")
        st = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled") and \
                    h.endswith("per_issue_active.ratio"):
                try:
                    st.append((h, float(v[0])))
                except ValueError:
                    pass
        for h, v in sorted(st, key=lambda x: -x[1])[:8]:
            print(f"  stall {h.split('stalled_')[1].split('_per')[0]} = {v:.2f}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if top and len(rows) > 2:
        hdr = rows[1]
        data = rows[2:]
        i_src = hdr.index("Source")
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        data = [r for r in data if len(r) > i_s and r[i_s].replace(".", "").isdigit()]
        tot = sum(float(r[i_s] or 0) for r in data)
        print(f"  sampled stalls: {tot:.0f}")
        for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]:
            print(f"   {float(r[i_s]) / tot * 100:5.1f}%  {r[i_src].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
