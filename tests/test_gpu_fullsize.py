"""Full-size parity at the BASELINE configs that fit one GPU, in the launch configuration bench.py
times (same fused kernel, 148 persistent CTAs), at the dual point the solver actually reaches (AGD
with gamma continuation + Jacobi, the bench schedule):

* configs[1] 1M x 10k, ~1e8 nnz, simplex;
* configs[3] 10M x 10k, ~1e9 nnz, two constraint families, box-cut (0 <= x <= 1, sum <= 3);
* configs[4] 330M sources x 100k, ~2e9 nnz, power-law block lengths 1..10k, simplex
  (lambda too large for shared memory: the global-lambda kernel variant; blocks >= 256 entries
  on the multi-warp path).

Checks:
* sampled outputs: x*(mu) of 3000 random sources (and the 200 longest blocks) recomputed one by
  one by the oracle projection;
* properties that hold at any size: the gradient equals A x - b for the x the kernel produced
  (scatter check), the dual value equals c^T x + gamma/2 ||x||^2 + mu^T (A x - b), every block of
  x lies in its polytope, nnz(x) is the count of positive x.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from oracle.projection import project  # noqa: E402
from paper_2603_04621_b200 import DL_PROJ_BOXCUT, DL_PROJ_SIMPLEX, MatchingProblem  # noqa: E402
from synth.matching import CONFIGS, generate  # noqa: E402

# workload -> (projection kind, r, u, solver iterations before the check)
WORKLOADS = {
    "1M_x_10k": (DL_PROJ_SIMPLEX, 1.0, np.inf, 1500),
    "multifamily_boxcut": (DL_PROJ_BOXCUT, 3.0, 1.0, 300),
    "powerlaw": (DL_PROJ_SIMPLEX, 1.0, np.inf, 200),
}


@pytest.fixture(scope="module", params=list(WORKLOADS))
def full(request):
    name = request.param
    kind, r, u, iters = WORKLOADS[name]
    inst = generate(CONFIGS[name], threads=16)
    gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=(1.0 if np.isinf(u) else u))
    gp.set_jacobi(gp.row_sqnorms())
    gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
    gp.solve(iters)
    gp.sync()
    yield name, inst, gp
    gp.close()


@pytest.mark.parametrize("gamma", [0.01, 0.16])
def test_fullsize_sampled_and_properties(full, gamma):
    name, inst, gp = full
    kind, r, u, _ = WORKLOADS[name]
    _, l2 = gp.dual()
    mu32 = l2.astype(np.float32)
    mu_t = torch.from_numpy(mu32).cuda()
    grad, obj = gp.dual_grad(mu_t, gamma)
    x = gp.primal(mu_t, gamma)
    torch.cuda.synchronize()
    grad, obj = grad.cpu().numpy(), obj.cpu().numpy()
    x = x.cpu().numpy()
    del mu_t
    rp, dest = inst.row_ptr, inst.dest
    m, J = inst.num_families, inst.num_dests
    mu = mu32.astype(np.float64)
    lens = np.diff(rp)
    # sampled blocks (random + the longest), one by one through the oracle projection
    rng = np.random.default_rng(11)
    sample = np.concatenate([rng.choice(inst.num_sources, 3000, replace=False), np.argsort(lens)[-200:]])
    for i in sample:
        sl = slice(rp[i], rp[i + 1])
        if sl.stop == sl.start:
            continue
        d = dest[sl]
        s = inst.c[sl].astype(np.float64)
        for f in range(m):
            s = s + inst.a[f, sl].astype(np.float64) * mu[f * J + d]
        np.testing.assert_allclose(x[sl], project(kind, -s / gamma, r, u), atol=2e-6, rtol=0)
    # polytope membership everywhere
    nz = lens > 0
    sums = np.add.reduceat(x, rp[:-1][nz], dtype=np.float64)
    assert np.all(x >= 0)
    over = np.flatnonzero(sums > r * (1 + 1e-5))
    if over.size:  # report the worst block against the oracle projection
        b = over[np.argmax(sums[over])]
        i = np.flatnonzero(nz)[b]
        sl = slice(rp[i], rp[i + 1])
        s = inst.c[sl].astype(np.float64)
        for f in range(m):
            s = s + inst.a[f, sl].astype(np.float64) * mu[f * J + dest[sl]]
        ref = project(kind, -s / gamma, r, u)
        import os
        os.makedirs("gpurun_out", exist_ok=True)
        np.savez(f"gpurun_out/fullsize_fail_{name}_{gamma}.npz", c=inst.c[sl], a=inst.a[:, sl], dest=dest[sl],
                 mu=mu32[[f * J + j for f in range(m) for j in dest[sl]]].reshape(m, -1), gamma=gamma, r=r, u=u,
                 x=x[sl], source=i)
        pytest.fail(f"{over.size} blocks with sum x > r; worst source {i} (len {lens[i]}): sum {sums[b]!r}, "
                    f"oracle sum {ref.sum()!r}, max |x - oracle| {np.max(np.abs(x[sl] - ref)):.3g}, "
                    f"x {x[sl][x[sl] > 0][:12]}, oracle {ref[ref > 0][:12]}")
    if np.isfinite(u):
        assert np.all(x <= u * (1 + 1e-6))
    # scatter: gradient == A x - b for the produced x (x output is fp32: tolerance from that rounding)
    x64 = x.astype(np.float64)
    pos = np.flatnonzero(x64 > 0)
    xp, dp = x64[pos], dest[pos]
    c = inst.c[pos].astype(np.float64)
    Ax = np.empty(m * J)
    absAx = np.empty(m * J)
    for f in range(m):
        af = inst.a[f, pos].astype(np.float64)
        Ax[f * J:(f + 1) * J] = np.bincount(dp, weights=af * xp, minlength=J)
        absAx[f * J:(f + 1) * J] = np.bincount(dp, weights=np.abs(af) * xp, minlength=J)
    np.testing.assert_array_less(np.abs(grad - (Ax - inst.b)), 1e-6 * (absAx + np.abs(inst.b)) + 1e-9)
    # objective terms
    cx = float(c @ xp)
    reg = 0.5 * gamma * float(xp @ xp)
    g = cx + reg + float(mu @ (Ax - inst.b))
    assert abs(obj[1] - cx) <= 1e-6 * float(np.abs(c) @ xp)
    assert abs(obj[2] - reg) <= 1e-5 * abs(reg) + 1e-9
    assert abs(obj[0] - g) <= 1e-6 * (float(np.abs(c) @ xp) + abs(reg) + float(np.abs(mu) @ (absAx + np.abs(inst.b))))
    assert obj[3] == pos.size
