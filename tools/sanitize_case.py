"""Small MSP-GMRES cases run under compute-sanitizer by tests/test_gpu_sanitizer.py:
a full solve (graph replay and direct launches), one MSP application and the single-step
entry points, on C1 (no AMG level) / a small C2 (several AMG levels, ABMC blocks)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import gen  # noqa: E402
from paper_2208_08594_b200 import MspSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
p = gen.make_config(name, **({} if name == "C1" else dict(nx=14, ny=12, nz=4)))
for kw in (dict(), dict(use_graphs=0, orth=0)):
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], coarsest_max_dof=60, **kw)
    b = torch.from_numpy(p["rhs"]).cuda()
    r = s.solve(b, tol=1e-8)
    assert r["final_rel"] <= 1e-8, r["final_rel"]
    N = p["n"] * p["b"]
    g = torch.from_numpy(gen.random_vector(N, 1)).cuda()
    w = torch.zeros_like(g)
    s.apply(g, w)
    s.bilu_forward(g, w)
    s.bilu_backward(g, w)
    s.pcol_residual(g, g[:p["n"]].contiguous(), w)
    s.restrict_pressure(g, torch.zeros(p["n"], dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    s.close()
del b, g, w
torch.cuda.empty_cache()
print("sanitize case ok", name, r["iters"])
