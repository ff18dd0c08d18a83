"""Candidate statistics at an AGD state (diagnostic): per block, the window count T = #{s - s_min <
gamma r}, the count after one Michelot step in the window, the min-2 window, and K* = #{x > 0}.

    python scripts/cand_hist.py CONFIG [num_sources] [iters]
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_04621_b200 import MatchingProblem
from synth.matching import CONFIGS, generate

name = sys.argv[1]
n_src = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[name].num_sources
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2500
cfg = dataclasses.replace(CONFIGS[name], num_sources=n_src)
inst = generate(cfg, threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
gp.solve(iters)
mu = gp.point().astype(np.float64)
gp.close()
gamma = 0.01
s = inst.c.astype(np.float64) + inst.a[0].astype(np.float64) * mu[inst.dest]
lens = np.diff(inst.row_ptr)
nz = lens > 0
starts = inst.row_ptr[:-1][nz]
src = np.repeat(np.arange(nz.sum()), lens[nz])
smin = np.minimum.reduceat(s, starts)
d = (s - smin[src]) / gamma
win = d < 1.0
T = np.bincount(src, weights=win, minlength=smin.size)
S = np.bincount(src, weights=np.where(win, d, 0), minlength=smin.size)
phi1 = (1.0 + S) / np.maximum(T, 1)
T1 = np.bincount(src, weights=win & (d < phi1[src]), minlength=smin.size)
# second smallest
big = np.where(d > 0, d, np.inf)
d2 = np.minimum.reduceat(big, starts)
w2 = np.minimum(1.0, (1.0 + np.where(np.isfinite(d2), d2, 1.0)) / 2)
T2 = np.bincount(src, weights=d < w2[src], minlength=smin.size)
# exact K*: Michelot to convergence on the window
phi = phi1.copy()
for _ in range(60):
    inn = win & (d < phi[src])
    c = np.bincount(src, weights=inn, minlength=smin.size)
    sm = np.bincount(src, weights=np.where(inn, d, 0), minlength=smin.size)
    phi = (1.0 + sm) / np.maximum(c, 1)
phi = np.minimum(phi, -smin / gamma)
K = np.bincount(src, weights=d < phi[src], minlength=smin.size)
for nm, v in (("T window", T), ("T after 1 Michelot step", T1), ("T min-2 window", T2), ("K* positive", K)):
    q = np.percentile(v, [50, 90, 99, 99.9])
    print(f"{name} {nm:26s} mean {v.mean():6.2f}  p50/90/99/99.9 {q}  max {v.max():.0f}  mean T^2 {np.mean(v**2):.1f}")
