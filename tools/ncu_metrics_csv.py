"""Per-launch summary of an ncu --set full report: time, DRAM bytes, achieved DRAM TB/s,
occupancy, registers, L2 hit rate, issue activity (one CSV row per profiled launch).

    python tools/ncu_metrics_csv.py gpurun_out/prof_full_r01.ncu-rep > profiles/r01/ncu_full_set_metrics.csv
"""
import csv
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--print-units", "base", "--metrics", ",".join(KEEP)],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
idx = [h.index("Kernel Name")] + [h.index(k) for k in KEEP]
w = csv.writer(sys.stdout)
w.writerow(["kernel"] + KEEP + ["dram_TBps"])
for r in rows[2:]:
    t, rd, wr = (float(r[h.index(k)].replace(",", "")) for k in KEEP[:3])     # ns, bytes, bytes (base units)
    w.writerow([r[idx[0]][:80]] + [r[i] for i in idx[1:]] + [f"{(rd + wr) / t / 1e3:.2f}" if t else ""])
