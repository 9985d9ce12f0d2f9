"""Print ms/step, per-kernel and per-level times of bench lines (tools/gpu_ab_*.sh output)."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_*.json")):
    try:
        d = json.loads(open(f).read())
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    ks = " ".join(f"{k}={v['ms'] * 1e3:.1f}us" for k, v in d.get("kernels", {}).items())
    print(f"{f}: {d['ms_per_step']:.3f} ms/step iters={d['config'].get('iterations')} {ks}")
    if d.get("vcycle_levels"):
        print("    levels:", " ".join(f"L{v.get('level')}={v.get('ms', 0) * 1e3:.1f}us" for v in d["vcycle_levels"]))
