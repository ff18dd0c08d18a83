"""First fused pass at a new AGD point via the solver eval vs the standalone entry (diagnostic;
DUALIP_TRACE=1)."""
import os
import sys

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
grad, obj = gp.new_grad_buffers()
mu = torch.empty(gp.n, dtype=torch.float32, device="cuda")


def span(tag):
    gp.sync()
    raw = L.dl_debug_trace(gp.h)
    tr = raw[:5 * gp.info["ctas"]].reshape(-1, 5)
    print(f"{tag:40s} {(tr[:, 3].max() - tr[:, 1].min()) / 1e3:7.1f} us  tiles/CTA {tr[:, 4].min()}..{tr[:, 4].max()}",
          flush=True)


E = lambda: L.dl_agd_eval(gp.h)
S = lambda: L.dl_dual_step(gp.h)


def D():
    L.dl_agd_point(gp.h, mu)
    gp.dual_grad(mu, 0.01, out=(grad, obj))


for k in range(3):
    D(); span(f"{k}: D first at the point")
    E(); span(f"{k}: E second at the point")
    S()
    E(); span(f"{k}: E first at the point")
    D(); span(f"{k}: D second at the point")
    S()
    E(); span(f"{k}: E first at the point")
    S()
