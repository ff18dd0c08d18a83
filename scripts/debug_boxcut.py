import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.matching import GenConfig, generate
from oracle.dual import Problem, primal, BOXCUT
from paper_2603_04621_b200 import MatchingProblem
cfg = GenConfig(num_sources=1500, num_dests=20000, length_law="powerlaw", max_len=6000, powerlaw_alpha=1.5, seed=24)
inst = generate(cfg)
gp = MatchingProblem.from_instance(inst, kind=1, r=4.0, u=0.6)
P = Problem.from_instance(inst, kind=BOXCUT, r=4.0, u=0.6)
rng = np.random.default_rng(hash("boxcut_powerlaw") % 2**32)
lens = np.diff(inst.row_ptr)
for lam in (np.zeros(gp.n, np.float32), (rng.exponential(2.0/np.sqrt(inst.nnz/inst.num_dests), gp.n)*(rng.random(gp.n)<0.8)).astype(np.float32)):
    for gamma in (0.01, 0.16, 1.0):
        x = gp.primal(torch.from_numpy(lam).cuda(), gamma); torch.cuda.synchronize(); x = x.cpu().numpy()
        xo = primal(P, lam.astype(np.float64), gamma)
        err = np.abs(x - xo)
        src = np.repeat(np.arange(lens.size), lens)
        be = np.zeros(lens.size); np.maximum.at(be, src, err)
        bad = np.argsort(-be)[:5]
        print(f"gamma {gamma} max err {err.max():.3e}; worst blocks:", [(int(i), int(lens[i]), f"{be[i]:.2e}") for i in bad])
        i = int(bad[0]); sl = slice(inst.row_ptr[i], inst.row_ptr[i+1])
        if be[i] > 1e-6:
            print("   gpu", np.round(x[sl][np.argsort(-xo[sl])][:10], 6), "sum", x[sl].sum())
            print("   orc", np.round(np.sort(xo[sl])[::-1][:10], 6), "sum", xo[sl].sum())
from oracle.dual import dual_eval, apply_A
for lam in (np.zeros(gp.n, np.float32), (rng.exponential(2.0/np.sqrt(inst.nnz/inst.num_dests), gp.n)*(rng.random(gp.n)<0.8)).astype(np.float32)):
    for gamma in (0.01, 0.16, 1.0):
        grad, obj = gp.dual_grad(torch.from_numpy(lam).cuda(), gamma); torch.cuda.synchronize()
        grad = grad.cpu().numpy()
        ev = dual_eval(P, lam.astype(np.float64), gamma)
        absAx = apply_A(P, np.abs(ev.x))
        tol = 1e-5 * (absAx + np.abs(P.b)) + 1e-12
        err = np.abs(grad - ev.grad)
        j = int(np.argmax(err / tol))
        print(f"gamma {gamma}: worst ratio {err[j]/tol[j]:.3f} at j={j}: gpu {grad[j]!r} orc {ev.grad[j]!r} Ax_orc {ev.Ax[j]!r} b {P.b[j]!r} absAx {absAx[j]!r}")
        sel = np.flatnonzero(P.dest == j)
        xs = ev.x[sel]; 
        print("    edges", sel.size, "x_orc nonzero", np.count_nonzero(xs), "max", xs.max() if xs.size else 0)
print("---- relative x errors")
for lam in (np.zeros(gp.n, np.float32), (rng.exponential(2.0/np.sqrt(inst.nnz/inst.num_dests), gp.n)*(rng.random(gp.n)<0.8)).astype(np.float32)):
    for gamma in (0.01, 0.16, 1.0):
        x = gp.primal(torch.from_numpy(lam).cuda(), gamma); torch.cuda.synchronize(); x = x.cpu().numpy().astype(np.float64)
        xo = primal(P, lam.astype(np.float64), gamma)
        rel = np.abs(x - xo) / np.maximum(np.abs(xo), 1e-3)
        e = int(np.argmax(rel)); i = int(np.searchsorted(inst.row_ptr, e, side='right') - 1)
        sl = slice(inst.row_ptr[i], inst.row_ptr[i+1])
        print(f"gamma {gamma}: worst rel {rel[e]:.2e} x {x[e]!r} xo {xo[e]!r} block {i} len {lens[i]} nnz(xo) {np.count_nonzero(xo[sl])} sum xo {xo[sl].sum():.6f} sum x {x[sl].sum():.6f} capped {np.sum(xo[sl] > 0.6 - 1e-12)}")
