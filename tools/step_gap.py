"""Host gap between Arnoldi steps: one C3 solve's device time vs the sum of its steps
(graph-replayed steps timed alone at j = 15 and 25, linear in j in between)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import gen  # noqa: E402
from paper_2208_08594_b200 import MspSolver  # noqa: E402

p = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"])
b = torch.from_numpy(p["rhs"]).cuda()
for _ in range(2):
    r = s.solve(b)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    r = s.solve(b)
torch.cuda.synchronize()
solve = (time.perf_counter() - t0) / 5 * 1e3
it = r["iters"]
s15 = s.time_kernel("arnoldi_step15", reps=20, flush=False)[0]
s25 = s.time_kernel("arnoldi_step25", reps=20, flush=False)[0]
slope = (s25 - s15) / 10
js = [j % 30 for j in range(it)]
est = sum(s15 + slope * (j - 15) for j in js)
print(f"iters {it}  solve {solve:.3f} ms (wall)  step15 {s15:.4f}  step25 {s25:.4f} ms  sum of steps {est:.3f} ms  "
      f"other (cycle ends + host gaps) {solve - est:.3f} ms = {(solve - est) / it * 1e3:.1f} us/iter")
