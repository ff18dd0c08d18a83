"""One fused dual-gradient launch of a (scaled) BASELINE workload at an AGD state, for ncu.

    ncu --nvtx --nvtx-include "fused/" ... python scripts/profile_config.py CONFIG [num_sources] [iters]
The projection of each workload is bench.WORKLOADS'; the instance keeps the workload's law
(lengths, destinations, families) with num_sources sources.
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import WORKLOADS
from paper_2603_04621_b200 import MatchingProblem
from synth.matching import CONFIGS, generate

name = sys.argv[1]
n_src = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[name].num_sources
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 500
cfg = dataclasses.replace(CONFIGS[name], num_sources=n_src)
_, kind, r, u = WORKLOADS[name][:4]
inst = generate(cfg, threads=16)
gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=u)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(iters)
gp.sync()
l1, l2 = gp.dual()
mu = torch.from_numpy(l2.astype(np.float32)).cuda()
grad, obj = gp.new_grad_buffers()
for _ in range(3):
    gp.dual_grad(mu, 0.01, out=(grad, obj))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(gp.stream)
for _ in range(10):
    gp.dual_grad(mu, 0.01, out=(grad, obj))
e1.record(gp.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
B = (8 + 4 * inst.num_families) * inst.nnz
print(f"{name} I={n_src} nnz={inst.nnz} after {iters} its: ms/eval={ms:.4f} GB/s={B / ms / 1e6:.1f} "
      f"nnz_x={obj[3].item():.0f} tiles={gp.info['num_tiles']} tile_cap={gp.info['tile_cap']} hot={gp.info['lambda_hot']}", flush=True)
torch.cuda.nvtx.range_push("fused")
gp.dual_grad(mu, 0.01, out=(grad, obj))
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
