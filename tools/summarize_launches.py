"""Summarise an ncu launch-list CSV (one full solve) into per-kernel shares and the
per-piece DRAM traffic used by bench.py's roofline.traffic (profiles/traffic.json)."""
import collections
import csv
import json
import sys

src, dst_txt, dst_json = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
    names[int(r[ii])] = r[ki].split("(")[0].replace("void mspk::", "").replace("void ", "")
tot = collections.defaultdict(float)
cnt = collections.Counter()
byt = collections.defaultdict(float)
for i, m in per.items():
    n = names[i]
    tot[n] += m.get("gpu__time_duration.sum", 0)
    cnt[n] += 1
    byt[n] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
T = sum(tot.values())
with open(dst_txt, "w") as f:
    f.write(f"# ncu launch list of one full C3 MSP-GMRES solve ({sum(cnt.values())} launches); "
            "cold-cache, serialised (compare SHARES)\n")
    f.write(f"# total kernel time {T / 1e6:.3f} ms\n")
    f.write("share%   total_ms  launches  avg_us  dram_GB/s  dram_MB/launch  kernel\n")
    for n, t in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"{t / T * 100:6.2f} {t / 1e6:9.3f} {cnt[n]:8d} {t / cnt[n] / 1e3:8.2f} "
                f"{byt[n] / t if t else 0:9.1f} {byt[n] / cnt[n] / 1e6:12.2f}  {n}\n")
pieces = {
    "a2_bsr_spmv": lambda n: n.startswith("bsr_spmv4c_kernel<0>") or n.startswith("bsr_spmv_kernel<4, 0>"),
    "a8_pcol_residual": lambda n: (n.startswith("bsr_spmv_kernel<4, 2>") or "pcol_resid4_kernel" in n
                                   or "pcol_resid_ell4_kernel" in n),
    "a9_bilu_apply": lambda n: n.startswith("bilu_block_kernel") or n.startswith("bilu_meta"),
}
out = {}
for key, pred in pieces.items():
    b = sum(byt[n] for n in byt if pred(n))
    c = sum(cnt[n] for n in cnt if pred(n))
    if key == "a9_bilu_apply":            # one BILU apply per MSP apply (one a3 launch each)
        c = sum(cnt[n] for n in cnt if n.startswith("restrict_pressure_kernel"))
    out[key] = b / c if c else None          # DRAM bytes per launch (per application)
out["_source"] = src
json.dump(out, open(dst_json, "w"), indent=1)
print(open(dst_txt).read()[:3000])
print(out)
