"""GPU AGD / solve parity (A4, A5): dl_solve against oracle.agd on the same seeded
instance, with and without Jacobi preconditioning and gamma continuation.

Both sides evaluate the gradient at mu_t = fl32(D lam2_t) (R7); the
only differences are reduction orders (fp64), so trajectories agree closely
until fp32 rounding of mu flips an ulp; the test bounds the relative gap in
g_t over the first iterations and in the final value."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from oracle.agd import AgdConfig, agd  # noqa: E402
from oracle.dual import Problem  # noqa: E402
from paper_2603_04621_b200 import MatchingProblem  # noqa: E402
from synth.matching import CONFIGS, GenConfig, generate  # noqa: E402


def run_both(inst, iters, cfg: AgdConfig):
    gp = MatchingProblem.from_instance(inst)
    if cfg.jacobi:
        gp.set_jacobi(gp.row_sqnorms())
    gp.agd_init(gamma0=cfg.gamma0, gamma_min=cfg.gamma_min or 0.0, halve_every=cfg.halve_every,
                use_jacobi=cfg.jacobi, max_step=cfg.max_step, init_step=cfg.init_step)
    gp.solve(iters)
    h = gp.history()
    l1, l2 = gp.dual()
    gp.close()
    tr = agd(Problem.from_instance(inst), iters, cfg)
    return h, (l1, l2), tr


@pytest.mark.parametrize("cfg", [AgdConfig(gamma0=0.01), AgdConfig(gamma0=0.01, jacobi=False),
                                 AgdConfig(gamma0=0.16, gamma_min=0.01, halve_every=25)])
def test_solve_trajectory_matches_oracle(cfg):
    inst = generate(CONFIGS["tiny"])
    iters = 300
    h, (l1, l2), tr = run_both(inst, iters, cfg)
    assert h.size == iters
    np.testing.assert_array_equal(h["iter"], np.arange(iters))
    np.testing.assert_allclose(h["gamma"], tr.gamma, rtol=0, atol=0)
    g_o = np.array(tr.g)
    # early iterations: the same point up to fp32 rounding flips of mu and fp32 thresholds
    np.testing.assert_allclose(h["g"][:50], g_o[:50], rtol=2e-6)
    np.testing.assert_allclose(h["eta"][:50], tr.eta[:50], rtol=1e-4)
    # whole run: same trajectory up to accumulated fp32 rounding of mu
    np.testing.assert_allclose(h["g"], g_o, rtol=1e-5)
    np.testing.assert_allclose(l1, tr.d * tr.lam1, rtol=1e-4, atol=1e-6 * np.abs(tr.d * tr.lam1).max())


def test_single_step_parity():
    inst = generate(GenConfig(num_sources=3000, num_dests=300, nnz_per_source=60, seed=40))
    h, _, tr = run_both(inst, 3, AgdConfig(gamma0=0.05, max_step=1e-2))
    np.testing.assert_allclose(h["g"], tr.g, rtol=1e-10)
    np.testing.assert_allclose(h["eta"], tr.eta, rtol=1e-10)
    np.testing.assert_allclose(h["gnorm"], tr.gnorm, rtol=1e-9)
    np.testing.assert_allclose(h["infeas"], tr.infeas, rtol=1e-9)


def test_solve_converges_like_oracle():
    """Reaching a 1e-3 relative dual gap takes the same number of iterations (+-2%)."""
    inst = generate(GenConfig(num_sources=300, num_dests=20, nnz_per_source=5, seed=11))
    cfg = AgdConfig(gamma0=0.01)
    h, _, tr = run_both(inst, 1500, cfg)
    ghat = max(tr.g)
    def first(gs):
        best = np.maximum.accumulate(np.asarray(gs))
        return int(np.flatnonzero(ghat - best <= 1e-3 * abs(ghat))[0])
    a, b = first(h["g"]), first(tr.g)
    assert abs(a - b) <= max(3, 0.02 * b), (a, b)


def test_reinit_rebuilds_the_solve_graph():
    """dl_agd_init after a graph-captured dl_solve (new history capacity, Jacobi switched on) must
    restart from lambda = 0 with the new buffers: the second run equals a fresh one."""
    inst = generate(CONFIGS["tiny"])
    cfg = AgdConfig(gamma0=0.01)
    gp = MatchingProblem.from_instance(inst)
    gp.agd_init(gamma0=0.01, use_jacobi=False, max_step=1e-3, init_step=1e-5, history_cap=64)
    gp.solve(40)                                   # captures the solve graph
    gp.set_jacobi(gp.row_sqnorms())
    gp.agd_init(gamma0=0.01, use_jacobi=True, max_step=1e-3, init_step=1e-5, history_cap=500)
    gp.solve(100)
    h = gp.history()
    gp.close()
    tr = agd(Problem.from_instance(inst), 100, cfg)
    assert h.size == 100
    np.testing.assert_allclose(h["g"], tr.g, rtol=1e-6)
