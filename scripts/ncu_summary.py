"""Summarise one ncu --set full capture (a .ncu-rep, or its `--page raw --csv` export) of a
generation kernel: the metrics the bench line and DESIGN.md quote, and the stall mix.

    python scripts/ncu_summary.py <prof.ncu-rep | raw.csv> [> profiles/rNN_ncu_full_<cfg>.txt]
"""
import csv
import subprocess
import sys

src = sys.argv[1]
if src.endswith(".csv"):
    text = open(src).read()
else:
    text = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                          text=True).stdout
r = list(csv.reader(text.splitlines()))
h, u, v = r[0], r[1], r[-1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"]
for k in keys:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]} {u[h.index(k)]}")
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((k, float(v[i].replace(",", ""))))
        except ValueError:
            pass
st.sort(key=lambda x: -x[1])
tot = sum(x[1] for x in st) or 1.0
print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100 * x / tot:.0f}%"
                           for k, x in st[:8]))
