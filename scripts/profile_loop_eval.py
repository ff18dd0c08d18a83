"""The 6th dl_agd_eval of a live [eval, step] loop after `iters` AGD iterations (nvtx "loop"), then one
standalone dl_dual_grad at the next point (nvtx "sa"), for ncu --replay-mode application.

    ncu --replay-mode application --cache-control none --nvtx --nvtx-include "loop/" ... python scripts/profile_loop_eval.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_04621_b200 import MatchingProblem
from paper_2603_04621_b200 import _lib as L
from synth.matching import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "1M_x_10k"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2500
inst = generate(CONFIGS[name], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(iters)
for k in range(6):
    if k == 5:
        torch.cuda.nvtx.range_push("loop")
    L.dl_agd_eval(gp.h)
    if k == 5:
        torch.cuda.nvtx.range_pop()
    L.dl_dual_step(gp.h)
gp.sync()
mu = torch.from_numpy(gp.point().astype(np.float32)).cuda()
grad, obj = gp.new_grad_buffers()
torch.cuda.nvtx.range_push("sa")
gp.dual_grad(mu, 0.01, out=(grad, obj))
torch.cuda.nvtx.range_pop()
gp.sync()
print("ok", flush=True)
