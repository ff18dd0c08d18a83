"""Candidate statistics of the fused kernel's fp32 filter along an AGD run (diagnostic)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.matching import CONFIGS, generate
from paper_2603_04621_b200 import MatchingProblem
inst = generate(CONFIGS["1M_x_10k"], threads=16)
gp = MatchingProblem.from_instance(inst)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
rp = inst.row_ptr; lens = np.diff(rp); src = np.repeat(np.arange(lens.size), lens)
a = inst.a[0].astype(np.float64); c = inst.c.astype(np.float64); d = inst.dest
done = 0
for target in (100, 300, 1000, 3000):
    gp.solve(target - done); done = target; gp.sync()
    l1, l2 = gp.dual()
    mu = l2.astype(np.float32).astype(np.float64)
    h = gp.history(); gamma = h["gamma"][-1]
    s = c + a * mu[d]
    smin = np.minimum.reduceat(s, rp[:-1])
    rel = s - smin[src]
    for W in (gamma,):
        cand = rel <= W * 1.000001 + 1e-6
        nc = np.bincount(src, weights=cand, minlength=lens.size)
        # per-lane (G=8 strided) max candidates
        lane = (np.arange(s.size) - rp[src]) % 8
        key = src * 8 + lane
        nl = np.bincount(key, weights=cand, minlength=lens.size * 8).reshape(-1, 8).max(axis=1)
        print(f"iter {target} gamma {gamma:.3g} nnz_x {h['nnz_x'][-1]:.0f}: cand/block mean {nc.mean():.2f} "
              f"p50 {np.median(nc):.0f} p90 {np.percentile(nc,90):.0f} p99 {np.percentile(nc,99):.0f} max {nc.max():.0f}; "
              f"lane max>3: {np.mean(nl>3)*100:.2f}% >1: {np.mean(nl>1)*100:.1f}%  T>=2: {np.mean(nc>=2)*100:.1f}%", flush=True)
