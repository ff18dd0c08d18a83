"""One fused dual-gradient launch at the converged AGD state of BASELINE configs[1] (for ncu).

    ncu --nvtx --nvtx-include "fused/" ... python scripts/profile_state.py [iters]
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.matching import CONFIGS, generate
from paper_2603_04621_b200 import MatchingProblem
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2510
inst = generate(CONFIGS["1M_x_10k"], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(iters); gp.sync()
l1, l2 = gp.dual()
mu = torch.from_numpy(l2.astype(np.float32)).cuda()
grad, obj = gp.new_grad_buffers()
for _ in range(3):
    gp.dual_grad(mu, 0.01, out=(grad, obj))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(gp.stream)
for _ in range(20):
    gp.dual_grad(mu, 0.01, out=(grad, obj))
e1.record(gp.stream); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"state after {iters} its: ms/eval={ms:.4f} GB/s={12*inst.nnz/ms/1e6:.1f} nnz_x={obj[3].item():.0f}", flush=True)
torch.cuda.nvtx.range_push("fused")
gp.dual_grad(mu, 0.01, out=(grad, obj))
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
