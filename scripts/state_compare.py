"""Diagnostic: cost of the fused pass at the AGD evaluation point vs the standalone entry.

    python scripts/state_compare.py [config] [iters]
Times dl_agd_eval (solver buffers, device gamma) and dl_dual_grad at the solver's evaluation point
(dl_agd_point) and at fl32 of dl_agd_dual's lambda2, and prints window-candidate statistics
(T = #{s - s_min < gamma r} per block) at both points.
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
gp.sync()
s = gp.stream


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


mu_pt = gp.point().astype(np.float32)
_, l2 = gp.dual()
mu_l2 = l2.astype(np.float32)
grad, obj = gp.new_grad_buffers()
print(f"{name} after {iters}: max|point - fl32(lam2)| = {np.max(np.abs(mu_pt - mu_l2)):.3e}", flush=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(s)
L.dl_agd_eval(gp.h)
ev[1].record(s)
torch.cuda.synchronize()
print(f"dl_agd_eval (one launch): {ev[0].elapsed_time(ev[1]):.4f} ms", flush=True)
print(f"dl_agd_eval x10: {timed(lambda: L.dl_agd_eval(gp.h)):.4f} ms", flush=True)
def loop_ms(pre, timed_fn, post, n=20):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for k in range(n):
        pre()
        evs[k][0].record(s)
        timed_fn()
        evs[k][1].record(s)
        post()
    torch.cuda.synchronize()
    return np.mean([a.elapsed_time(b) for a, b in evs[2:]])


nop = lambda: None
tq = torch.from_numpy(mu_pt).cuda()
L.dl_dual_step(gp.h)
print(f"loop [eval | step]: {loop_ms(nop, lambda: L.dl_agd_eval(gp.h), lambda: L.dl_dual_step(gp.h)):.4f} ms")
print(f"loop [dual_grad]: {loop_ms(nop, lambda: gp.dual_grad(tq, 0.01, out=(grad, obj)), nop):.4f} ms")
print(f"loop [dual_grad | step]: "
      f"{loop_ms(nop, lambda: gp.dual_grad(tq, 0.01, out=(grad, obj)), lambda: L.dl_dual_step(gp.h)):.4f} ms")
print(f"loop [step | dual_grad]: "
      f"{loop_ms(lambda: L.dl_dual_step(gp.h), lambda: gp.dual_grad(tq, 0.01, out=(grad, obj)), nop):.4f} ms")
acc_ptr, acc_n = L.dl_agd_accumulator(gp.h)


class _Arr:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


acc_t = torch.as_tensor(_Arr(acc_ptr, acc_n), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with torch.cuda.stream(s):
    print(f"loop [acc.zero_ | eval | step]: "
          f"{loop_ms(lambda: acc_t.add_(0.0), lambda: L.dl_agd_eval(gp.h), lambda: L.dl_dual_step(gp.h)):.4f} ms")
    print(f"loop [flush L2 | eval | step]: "
          f"{loop_ms(lambda: flush.fill_(1), lambda: L.dl_agd_eval(gp.h), lambda: L.dl_dual_step(gp.h)):.4f} ms")
    print(f"loop [flush L2 | dual_grad]: "
          f"{loop_ms(lambda: flush.fill_(1), lambda: gp.dual_grad(tq, 0.01, out=(grad, obj)), nop):.4f} ms")
g_solver = float(gp.history()["gamma"][-1])
print(f"solver gamma {g_solver!r} vs 0.01 {0.01!r}", flush=True)
tp = torch.from_numpy(mu_pt).cuda()
print(f"dl_dual_grad at point, solver gamma: {timed(lambda: gp.dual_grad(tp, g_solver, out=(grad, obj))):.4f} ms",
      flush=True)
for nm, mu in (("point", mu_pt), ("lam2", mu_l2)):
    t = torch.from_numpy(mu).cuda()
    ms = timed(lambda: gp.dual_grad(t, 0.01, out=(grad, obj)))
    print(f"dl_dual_grad at {nm}: {ms:.4f} ms  nnz_x {obj[3].item():.0f}", flush=True)
    m64 = mu.astype(np.float64)
    sc = inst.c.astype(np.float64) + inst.a[0].astype(np.float64) * m64[inst.dest]
    lens = np.diff(inst.row_ptr)
    nz = lens > 0
    starts = inst.row_ptr[:-1][nz]
    src = np.repeat(np.arange(nz.sum()), lens[nz])
    smin = np.minimum.reduceat(sc, starts)
    d = (sc - smin[src]) / 0.01
    T = np.bincount(src, weights=d < 1.0, minlength=smin.size)
    q = np.percentile(T, [50, 90, 99, 99.9])
    print(f"   window T: mean {T.mean():.2f} p50/90/99/99.9 {q} max {T.max():.0f}; blocks with T > 32: "
          f"{np.mean(T > 32):.4f}", flush=True)
