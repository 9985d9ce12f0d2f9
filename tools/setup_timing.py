"""SETUP phase timing (msp_setup, NEXT-2): two setups of the same matrix in one process
(the second is what repeated ASMSP rebuilds pay), with the per-phase breakdown
(MSP_SETUP_VERBOSE) on stderr."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401
import gen  # noqa: E402
from paper_2208_08594_b200 import MspSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = gen.make_config(cfg)
if "--device" in sys.argv:                 # BSR arrays already on the GPU (msp_bsr device >= 0)
    p = dict(p, row_ptr=torch.from_numpy(p["row_ptr"]).int().cuda(), col=torch.from_numpy(p["col"]).int().cuda(),
             val=torch.from_numpy(p["val"]).double().cuda())
    torch.cuda.synchronize()
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2):
    t0 = time.time()
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"])
    print(f"{cfg} setup {k}: wall {time.time() - t0:.3f} s, library {s.stats()['last_setup_seconds']:.3f} s",
          file=sys.stderr, flush=True)
    s.close()
