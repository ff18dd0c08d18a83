"""Per-CTA start/end of the fused pass in the live solver loop vs after a spacer kernel (diagnostic).

    DUALIP_TRACE=1 python scripts/trace_eval.py [config] [iters]
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
spacer = torch.zeros(16, device="cuda")


def show(tag, raw):
    tr = raw[:5 * gp.info["ctas"]].reshape(-1, 5)
    ch = raw[5 * gp.info["ctas"]:]
    t0 = tr[:, 1].min()
    nch = (gp.info["num_tiles"] - gp.info["num_big_tiles"]) // 8
    tc = (ch[:nch].astype(np.int64) - int(t0)) / 1e3
    dec = [np.percentile(tc[int(nch * q / 10):int(nch * (q + 1) / 10)], 50) for q in range(10)]
    st = (tr[:, 1] - t0) / 1e3
    stg = (tr[:, 2] - t0) / 1e3
    en = (tr[:, 3] - t0) / 1e3
    print(f"{tag}: span {en.max():.1f} us; CTA start min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f}; "
          f"staged med {np.median(stg):.1f}; end min/med/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}; "
          f"tiles min/med/max {tr[:, 4].min()}/{int(np.median(tr[:, 4]))}/{tr[:, 4].max()}; "
          f"distinct SMs {len(set(tr[:, 0].tolist()))}", flush=True)
    print("   median completion (us) of each tenth of the chunk list:", np.round(dec, 1).tolist(), flush=True)


for k in range(3):  # the live loop: eval, step, eval, ... (host ahead of the GPU); trace of the last eval
    for _ in range(6):
        L.dl_agd_eval(gp.h)
        L.dl_dual_step(gp.h)
    L.dl_agd_eval(gp.h)
    gp.sync()
    show(f"eval after step {k}", L.dl_debug_trace(gp.h))
    if k == 0:
        raw = L.dl_debug_trace(gp.h)
        np.save("gpurun_out/r02_chunk_times_slow.npy", raw)
    L.dl_dual_step(gp.h)
with torch.cuda.stream(s):
    for k in range(3):
        for _ in range(6):
            spacer.add_(1.0)
            L.dl_agd_eval(gp.h)
            L.dl_dual_step(gp.h)
        spacer.add_(1.0)
        L.dl_agd_eval(gp.h)
        gp.sync()
        show(f"eval after spacer {k}", L.dl_debug_trace(gp.h))
        L.dl_dual_step(gp.h)
acc_ptr, acc_n = L.dl_agd_accumulator(gp.h)


class _Arr:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


acc_t = torch.as_tensor(_Arr(acc_ptr, acc_n), device="cuda")
hbuf = torch.zeros(16).pin_memory()
dbuf = torch.zeros(16, device="cuda")
import ctypes
import glob
_rt = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                         "libcudart.so*"))[0])
_rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
g2b, o2b = gp.new_grad_buffers()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fsum = torch.empty(1, dtype=torch.int64, device="cuda")
mu_dev = torch.empty(gp.n, dtype=torch.float32, device="cuda")
for nm, pre in (("dl_agd_point into device memory", lambda: L.dl_agd_point(gp.h, mu_dev)),
                ("dl_agd_point into host memory", lambda: gp.point()),
                ("L2 flush by a 256 MB write", lambda: flush.fill_(1)),
                ("acc.add_(0)", lambda: acc_t.add_(0.0)),
                ("cudaMemsetAsync 64 B", lambda: _rt.cudaMemsetAsync(dbuf.data_ptr(), 0, 64, s.cuda_stream)),
                ("cudaMemsetAsync acc", lambda: _rt.cudaMemsetAsync(acc_ptr, 0, 8 * acc_n, s.cuda_stream)),
                ("finalize (dl_agd_gradient)", lambda: L.dl_agd_gradient(gp.h, g2b, o2b))):
    with torch.cuda.stream(s):
        for _ in range(6):
            pre()
            L.dl_agd_eval(gp.h)
            L.dl_dual_step(gp.h)
        pre()
        L.dl_agd_eval(gp.h)
        gp.sync()
        show(f"eval after {nm}", L.dl_debug_trace(gp.h))
        L.dl_dual_step(gp.h)
mu = torch.from_numpy(gp.point().astype(np.float32)).cuda()
grad, obj = gp.new_grad_buffers()
gp.dual_grad(mu, 0.01, out=(grad, obj))
gp.sync()
show("A dual_grad at mu_T", L.dl_debug_trace(gp.h))
o1 = obj.cpu().numpy().copy()
L.dl_agd_eval(gp.h)
gp.sync()
show("B eval at mu_T", L.dl_debug_trace(gp.h))
g2, o2 = gp.new_grad_buffers()
L.dl_agd_gradient(gp.h, g2, o2)
gp.dual_grad(mu, 0.01, out=(grad, obj))
gp.sync()
show("C dual_grad at mu_T", L.dl_debug_trace(gp.h))
print("obj dual_grad", o1, "obj eval", o2.cpu().numpy(), flush=True)
print("acc", hex(acc_ptr), flush=True)
h = gp.history()
print("last history g/nnz_x/t:", h["g"][-1], h["nnz_x"][-1], len(h), flush=True)
