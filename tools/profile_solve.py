"""Profiling driver: C3 setup + one warm solve (captures the CUDA graphs), then the
profiled region (cudaProfilerStart/Stop) = one full MSP-GMRES solve.  Used with
`ncu --profile-from-start off`."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2208_08594_b200 import MspSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--kernel", default=None, help="time_kernel kind instead of a solve")
ap.add_argument("--orth", type=int, default=None, help="msp_config.orth (default: library default)")
a = ap.parse_args()
p = gen.make_config(a.config)
s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"],
              **({} if a.orth is None else dict(orth=a.orth)))
b = torch.from_numpy(p["rhs"]).cuda()
x = torch.zeros_like(b)
r = s.solve(b, x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.solves):
    if a.kernel:
        s.time_kernel(a.kernel, reps=2)
    else:
        x.zero_()
        r = s.solve(b, x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iters", r["iters"], "launches", s.kernel_launches())
