"""Quick timing probe of the fused pass on BASELINE configs[1] (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth.matching import CONFIGS, generate
from paper_2603_04621_b200 import MatchingProblem
t0 = time.time()
inst = generate(CONFIGS["1M_x_10k"], threads=16)
print("gen", time.time() - t0, inst.nnz, flush=True)
gp = MatchingProblem.from_instance(inst)
print(gp.info, flush=True)
rng = np.random.default_rng(0)
lam = torch.from_numpy((rng.exponential(0.02, gp.n)).astype(np.float32)).cuda()
grad, obj = gp.new_grad_buffers()
QUICK = os.environ.get("PROBE_QUICK")
if QUICK:
    for _ in range(3):
        gp.dual_grad(lam, 0.01, out=(grad, obj))
    torch.cuda.synchronize(); sys.exit(0)
for g in (0.01, 0.16):
    for _ in range(3):
        gp.dual_grad(lam, g, out=(grad, obj))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(gp.stream)
    N = 20
    for _ in range(N):
        gp.dual_grad(lam, g, out=(grad, obj))
    e1.record(gp.stream); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / N
    print(f"gamma={g} ms/eval={ms:.4f} nnz/s={inst.nnz/ms*1e3:.3e} GB/s={12*inst.nnz/ms/1e6:.1f} obj={obj.cpu().numpy()}", flush=True)
gp.agd_init(gamma0=0.01)
gp.set_jacobi(gp.row_sqnorms())
gp.agd_init(gamma0=0.01)
torch.cuda.synchronize(); t=time.time()
gp.solve(200); gp.sync()
print("solve 200 its s", time.time()-t)
h = gp.history(); print(h["g"][[0,1,10,50,100,199]], h["eta"][[0,1,199]], h["nnz_x"][-1])
