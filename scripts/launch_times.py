"""Per-kernel device times of the solver step (for ncu --metrics gpu__time_duration.sum):
solve(iters) then `n` stream-launched iterations [eval, step] inside an nvtx range "steps"."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import WORKLOADS
from paper_2603_04621_b200 import MatchingProblem
from paper_2603_04621_b200 import _lib as L
from synth.matching import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "1M_x_10k"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2500
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5
_, kind, r, u = WORKLOADS[name][:4]
inst = generate(CONFIGS[name], threads=16)
gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=u)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(iters)
gp.sync()
torch.cuda.nvtx.range_push("steps")
for _ in range(n):
    L.dl_agd_eval(gp.h)
    L.dl_dual_step(gp.h)
gp.sync()
torch.cuda.nvtx.range_pop()
