"""Michelot iteration counts from the all-candidates start at the converged AGD state (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.matching import CONFIGS, generate
from paper_2603_04621_b200 import MatchingProblem
inst = generate(CONFIGS["1M_x_10k"], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(3000); gp.sync()
l1, l2 = gp.dual()
mu = l2.astype(np.float32).astype(np.float64)
rp = inst.row_ptr; a = inst.a[0].astype(np.float64); c = inst.c.astype(np.float64); d = inst.dest
g = 0.01; r = 1.0
its = []; cands = []; act = []
for i in range(0, 1000000, 50):
    s = c[rp[i]:rp[i+1]] + a[rp[i]:rp[i+1]] * mu[d[rp[i]:rp[i+1]]]
    dd = (s - s.min()) / g
    C = np.sort(dd[dd <= r * 1.000001 + 1e-4])
    cands.append(C.size)
    phi_free = -s.min() / g
    if phi_free <= r and np.maximum(phi_free - dd, 0).sum() <= r:
        its.append(0); act.append(int((phi_free - dd > 0).sum())); continue
    S = C.size; phi = (r + C.sum()) / S; n = 1; prev = S
    while True:
        m = C < phi; k = int(m.sum())
        n += 1
        if k == prev: break
        prev = k; phi = (r + C[m].sum()) / k
    its.append(n); act.append(prev)
its = np.array(its); cands = np.array(cands); act = np.array(act)
print("cands mean", cands.mean(), "active mean", act.mean(), "iters mean", its.mean(), "p90", np.percentile(its, 90), "max", its.max())
# warp max over 4 consecutive blocks
w = its[: len(its) // 4 * 4].reshape(-1, 4).max(axis=1)
print("warp(4 groups) max iters mean", w.mean())
