"""Per-launch table of the a9 color phases from tools/gpu_bilu_launches.sh output."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    byid = collections.OrderedDict()
    for r in rows:
        byid.setdefault((r["ID"], r["Kernel Name"].split("(")[0]), {})[r["Metric Name"]] = r["Metric Value"]
    items = [kv for kv in byid.items() if "bilu" in kv[0][1]][-15:]
    print("#", path)
    tot_t = tot_b = 0.0
    for (i, name), m in items:
        d = float(m["gpu__time_duration.sum"].replace(",", "")) / 1e3
        rb = float(m["dram__bytes_read.sum"].replace(",", "")) / 1e6
        wb = float(m["dram__bytes_write.sum"].replace(",", "")) / 1e6
        tot_t += d; tot_b += rb + wb
        print(f"{name[-40:]:40s} grid {m['launch__grid_size']:>6s} {d:7.1f} us {rb + wb:8.1f} MB {(rb + wb) / d:5.2f} TB/s "
              f"warps {float(m['sm__warps_active.avg.pct_of_peak_sustained_active']):5.1f}% issue {float(m['smsp__issue_active.avg.pct_of_peak_sustained_active']):5.1f}%")
    print(f"# total {tot_t:.1f} us, {tot_b:.1f} MB, {tot_b / tot_t:.2f} TB/s")
