"""Writes tests/golden/oracle_<cfg>.json: the CPU oracle's MSP-GMRES result on a full-size
workload (default C3: SPE10-shaped 60x220x85, nc=3; C4: nc=6), tol 1e-6, GMRES(30).  Calls only oracle/ and
gen/ (seeded inputs).  Takes a few minutes single-threaded.
Optional second argument: pressure smoother (0 PGS-MC default, 1 PJAC-NO, 2 PGS-NO with
K = 32; reading R13) -> oracle_<cfg>_sm<k>.json.  The GMRES orthogonalisation of these
reference runs is CGS2 (orth=0, the textbook form, R8); the product's default DCGS2 (R14)
builds the same basis in exact arithmetic."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import gen      # noqa: E402
import oracle   # noqa: E402

CFG = sys.argv[1] if len(sys.argv) > 1 else "C3"
SM = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = gen.make_config(CFG)
t0 = time.time()
M = oracle.Msp(p["row_ptr"], p["col"], p["val"], smoother=SM, gs_chunk=32, orth=0)
t1 = time.time()
r = M.solve(p["rhs"], tol=1e-6, restart=30, maxit=1000)
t2 = time.time()
out = dict(config=CFG, smoother=SM, gs_chunk=32, orth=0, tol=1e-6, restart=30, iters=r["iters"], final_rel=r["final_rel"],
           hist=r["hist"].tolist(), status=r["status"], levels=M.info(),
           oracle_setup_s=t1 - t0, oracle_solve_s=t2 - t1, cores=1)
name = f"oracle_{CFG.lower()}.json" if SM == 0 else f"oracle_{CFG.lower()}_sm{SM}.json"
json.dump(out, open(os.path.join(HERE, name), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "hist"}))
