"""ASMSP over a synthetic Newton sequence: for each threshold
mu, run the sequence A^(1..K) through msp_update (reuse iff It^(iota-1) <= mu)
and msp_solve, and report the paper's columns: SetupCalls, SetupRatio
(setup / (setup + solve) wall time), Iter (total GMRES iterations), Time (setup + solve).

  python tools/asmsp_sequence.py --config C4 --steps 6 --mu 0 10 30
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2208_08594_b200 import MspSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--mu", type=int, nargs="+", default=[0, 10, 30])
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--out", default=None)
a = ap.parse_args()

rows = []
for mu in a.mu:
    s = None
    it_prev = 0
    tot_setup = tot_solve = 0.0
    iters = []
    setups = 0
    for iota in range(1, a.steps + 1):
        p = gen.make_config(a.config, newton_step=iota - 1)
        t0 = time.perf_counter()
        if s is None:
            s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"])
            did = True
        else:
            did = s.update(p["row_ptr"], p["col"], p["val"], iota=iota, last_iterations=it_prev, mu=mu)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        setups += int(did)
        if did:
            tot_setup += t1 - t0
        else:
            tot_solve += t1 - t0                      # value refresh counts as solve phase
        b = torch.from_numpy(p["rhs"]).cuda()
        t2 = time.perf_counter()
        r = s.solve(b, tol=a.tol)
        torch.cuda.synchronize()
        tot_solve += time.perf_counter() - t2
        it_prev = r["iters"]
        iters.append(r["iters"])
        print(f"mu={mu} iota={iota} setup={did} iters={r['iters']} rel={r['final_rel']:.2e}", flush=True)
        del p, b
    st = s.stats()
    rows.append(dict(mu=mu, setup_calls=setups, setup_ratio=tot_setup / (tot_setup + tot_solve),
                     iterations=sum(iters), per_step=iters, time_seconds=tot_setup + tot_solve,
                     setup_seconds=tot_setup, solve_seconds=tot_solve,
                     solve_device_seconds=st["solve_seconds"], reuse_calls=st["reuse_calls"]))
    print(json.dumps(rows[-1]), flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
out = dict(config=a.config, steps=a.steps, tol=a.tol, rows=rows)
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out))
