"""Solver eval cost vs GPU idle time between iterations (diagnostic; DUALIP_TRACE=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_04621_b200 import MatchingProblem
from paper_2603_04621_b200 import _lib as L
from synth.matching import CONFIGS, generate

inst = generate(CONFIGS["1M_x_10k"], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(2500)
mode = sys.argv[1] if len(sys.argv) > 1 else "none"
grad, obj = gp.new_grad_buffers()
mu = torch.empty(gp.n, dtype=torch.float32, device="cuda")
L.dl_agd_point(gp.h, mu)
gp.sync()
if mode == "D":          # the wrapper: stream waits + dl_dual_grad
    gp.dual_grad(mu, 0.01, out=(grad, obj))
elif mode == "raw":      # dl_dual_grad alone, on the problem's stream
    L.dl_dual_grad(gp.h, mu, 0.01, grad, obj, 0)
elif mode == "waits":    # only the wrapper's stream waits
    cur = gp._in()
    gp._out(cur)
elif mode == "torchop":  # a torch kernel on torch's current stream
    mu.add_(0.0)
gp.sync()
torch.cuda.synchronize()
print("mode", mode, flush=True)


def span():
    raw = L.dl_debug_trace(gp.h)
    tr = raw[:5 * gp.info["ctas"]].reshape(-1, 5)
    return (tr[:, 3].max() - tr[:, 1].min()) / 1e3


for idle in (0.0, 0.001, 0.0):
    ts = []
    for k in range(8):
        L.dl_agd_eval(gp.h)
        gp.sync()
        ts.append(span())
        if idle:
            time.sleep(idle)
        L.dl_dual_step(gp.h)
    print(f"idle {idle * 1e3:6.1f} ms before each step: eval spans {np.round(ts, 0).tolist()}", flush=True)
