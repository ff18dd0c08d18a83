"""Per-iteration cost of the fused pass along the AGD trajectory (diagnostic, A/B of builds).

    DUALIP_LIB=path/to/libdualip.so python scripts/trajectory.py [iters] [config]
Prints the mean device time of dl_agd_eval (fused + deferred kernels) per window of iterations.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_04621_b200 import MatchingProblem
from paper_2603_04621_b200 import _lib as L
from synth.matching import CONFIGS, generate

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
name = sys.argv[2] if len(sys.argv) > 2 else "1M_x_10k"
inst = generate(CONFIGS[name], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5,
            history_cap=iters)
s = gp.stream
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
for t in range(iters):
    ev[t][0].record(s)
    L.dl_agd_eval(gp.h)
    ev[t][1].record(s)
    L.dl_dual_step(gp.h)
torch.cuda.synchronize()
ms = np.array([a.elapsed_time(b) for a, b in ev])
h = gp.history()
W = 250
print(f"{os.environ.get('DUALIP_LIB', 'in-tree')}: {name}, nnz {inst.nnz}, total eval ms {ms.sum():.1f}")
for w0 in range(0, iters, W):
    sl = slice(w0, min(iters, w0 + W))
    print(f"  it {w0:5d}-{sl.stop:5d}: eval ms mean {ms[sl].mean():.4f} max {ms[sl].max():.4f}  "
          f"nnz_x {h['nnz_x'][sl].mean():.3g}  gamma {h['gamma'][sl.stop - 1]:.3g}")
