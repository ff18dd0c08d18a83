"""One solver evaluation (dl_agd_eval, nvtx "agd") and one standalone evaluation at the same point
(dl_dual_grad, nvtx "sa") after `iters` AGD iterations, for ncu.

    ncu --nvtx --nvtx-include "agd/" --nvtx-include "sa/" ... python scripts/profile_eval.py [config] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import WORKLOADS
from paper_2603_04621_b200 import MatchingProblem
from paper_2603_04621_b200 import _lib as L
from synth.matching import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "1M_x_10k"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2500
_, kind, r, u, _ = WORKLOADS[name]
inst = generate(CONFIGS[name], threads=16)
gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=u)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(iters)
gp.sync()
mu = torch.from_numpy(gp.point().astype(np.float32)).cuda()
grad, obj = gp.new_grad_buffers()
torch.cuda.nvtx.range_push("agd")
L.dl_agd_eval(gp.h)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("sa")
gp.dual_grad(mu, 0.01, out=(grad, obj))
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", flush=True)
