"""Table 2 analog (NEXT-4): MSP-GMRES with PJAC-NO, PGS-NO and PGS-MC pressure
smoothers on one generated workload.  Per smoother: GMRES iterations to tol, device solve
time (CUDA events, mean of --reps solves after a warm-up solve), V-cycle time (graph
replay, L2 flushed).  Prints one JSON line per smoother (or writes --out).

    python tools/smoother_table.py --config C3 [--chunk 32] [--out file.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2208_08594_b200 import MspSolver  # noqa: E402

NAMES = {0: "PGS-MC", 2: "PGS-NO", 1: "PJAC-NO"}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--chunk", type=int, default=32)
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=None)
a = ap.parse_args()

p = gen.make_config(a.config)
b = torch.from_numpy(p["rhs"]).cuda()
rows = []
for sm in (1, 2, 0):
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], smoother=sm, gs_chunk=a.chunk)
    r = s.solve(b, tol=a.tol)
    t0 = s.stats()["solve_seconds"]
    for _ in range(a.reps):
        r = s.solve(b, tol=a.tol)
    solve_ms = (s.stats()["solve_seconds"] - t0) / a.reps * 1e3
    row = dict(config=a.config, smoother=NAMES[sm], gs_chunk=a.chunk if sm == 2 else None,
               iters=r["iters"], final_rel=r["final_rel"], solve_ms=round(solve_ms, 3),
               vcycle_ms=round(s.time_kernel("vcycle", reps=20)[0], 4),
               msp_apply_ms=round(s.time_kernel("msp_apply", reps=20)[0], 4))
    rows.append(row)
    print(json.dumps(row), flush=True)
    del s
    torch.cuda.empty_cache()
if a.out:
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)
