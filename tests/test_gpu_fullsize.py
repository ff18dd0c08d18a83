"""Full-size parity at BASELINE configs[1] (1M sources x 10k destinations, ~1e8 nnz), in the
launch configuration bench.py times (same fused kernel, 148 persistent CTAs), at the dual point
the solver actually reaches (AGD with gamma continuation + Jacobi, the bench schedule):

* sampled outputs: x*(mu) of 3000 random sources recomputed one by one by the oracle;
* properties that hold at any size: the gradient equals A x - b for the x the kernel
  produced (scatter check), the dual value equals c^T x + gamma/2 ||x||^2 + mu^T (A x - b),
  every block of x lies in its polytope.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from oracle.projection import project_simplex  # noqa: E402
from paper_2603_04621_b200 import MatchingProblem  # noqa: E402
from synth.matching import CONFIGS, generate  # noqa: E402


@pytest.fixture(scope="module")
def full():
    inst = generate(CONFIGS["1M_x_10k"], threads=16)
    gp = MatchingProblem.from_instance(inst)
    gp.set_jacobi(gp.row_sqnorms())
    gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
    gp.solve(1500)
    gp.sync()
    yield inst, gp
    gp.close()


@pytest.mark.parametrize("gamma", [0.01, 0.16])
def test_fullsize_sampled_and_properties(full, gamma):
    inst, gp = full
    _, l2 = gp.dual()
    mu32 = l2.astype(np.float32)
    mu_t = torch.from_numpy(mu32).cuda()
    grad, obj = gp.dual_grad(mu_t, gamma)
    x = gp.primal(mu_t, gamma)
    torch.cuda.synchronize()
    grad, obj, x = grad.cpu().numpy(), obj.cpu().numpy(), x.cpu().numpy().astype(np.float64)
    rp, dest = inst.row_ptr, inst.dest
    a = inst.a[0].astype(np.float64)
    c = inst.c.astype(np.float64)
    mu = mu32.astype(np.float64)
    # sampled blocks, one by one through the oracle projection
    rng = np.random.default_rng(11)
    for i in rng.choice(inst.num_sources, 3000, replace=False):
        sl = slice(rp[i], rp[i + 1])
        if sl.stop == sl.start:
            continue
        y = -(c[sl] + a[sl] * mu[dest[sl]]) / gamma
        np.testing.assert_allclose(x[sl], project_simplex(y, 1.0), atol=2e-6, rtol=0)
    # polytope membership everywhere
    lens = np.diff(rp)
    sums = np.add.reduceat(x, rp[:-1][lens > 0])
    assert np.all(x >= 0) and np.all(sums <= 1 + 1e-5)
    # scatter: gradient == A x - b for the produced x (x output is fp32: tolerance from that rounding)
    Ax = np.bincount(dest, weights=a * x, minlength=inst.num_dests)
    absAx = np.bincount(dest, weights=np.abs(a) * x, minlength=inst.num_dests)
    np.testing.assert_array_less(np.abs(grad - (Ax - inst.b)), 1e-6 * (absAx + np.abs(inst.b)) + 1e-9)
    # objective terms
    cx = float(c @ x)
    reg = 0.5 * gamma * float(x @ x)
    g = cx + reg + float(mu @ (Ax - inst.b))
    assert abs(obj[1] - cx) <= 1e-6 * abs(cx)
    assert abs(obj[2] - reg) <= 1e-5 * abs(reg) + 1e-9
    assert abs(obj[0] - g) <= 1e-6 * (abs(cx) + abs(reg) + float(np.abs(mu) @ (absAx + np.abs(inst.b))))
    assert obj[3] == np.count_nonzero(x > 0)
