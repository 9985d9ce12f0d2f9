"""Graph-replayed timing of MSP-GMRES pieces on a config (CUDA events, warm and cold L2)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import gen  # noqa
from paper_2208_08594_b200 import MspSolver  # noqa

p = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
variants = [("default", dict())]
for extra in sys.argv[2:]:
    if "=" in extra:
        variants.append((extra, dict()))
base_env = dict(os.environ)
for tag, kw in variants:
    os.environ.clear(); os.environ.update(base_env)
    if "=" in tag:
        for kv in tag.split(","):
            k, v = kv.split("=")
            if k.isupper():
                os.environ[k] = v                      # MSP_* environment switch
            else:
                kw[k] = int(v)                         # msp_config field (e.g. orth=2)
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], **kw)
    b = torch.from_numpy(p["rhs"]).cuda()
    r = s.solve(b)
    res = {}
    for k in ("arnoldi_step15", "arnoldi_step25", "cgs2_step25", "msp_apply", "vcycle", "bilu", "cgs2_step15", "a2_bsr_spmv", "a8_pcol_residual", "a4_pgs_sweep_l0", "a6_coarse_gemv", "bilu_spmv", "msp_apply_spmv", "spmv_orth15"):
        res[k + "_warm"] = s.time_kernel(k, reps=20, flush=False)[0]
        res[k + "_cold"] = s.time_kernel(k, reps=20, flush=True)[0]
    t0 = s.stats()["solve_seconds"]
    for _ in range(3):
        s.solve(b)
    res["solve_ms"] = (s.stats()["solve_seconds"] - t0) / 3 * 1e3
    print(tag, r["iters"], "kernels/step", s.stats()["kernels_per_iter"], flush=True)
    for k, v in res.items():
        print(f"  {k:28s} {v:9.4f} ms")
    s.close()
