"""GPU AGD / solve parity (A4, A5).

* Per-iterate pin (no oracle precision option): the solver is stepped through the C ABI, every
  dual point mu_t it visits is read back (dl_agd_point) together with the accumulated
  A x*(mu_t) and objective terms, and oracle.dual_eval -- the paper's fp64 dual
  -- is evaluated at that same mu_t: gradient and g(mu_t) must agree at the R12 tolerance at
  every iterate, so the whole GPU trajectory is checked without the oracle copying any kernel
  rounding.
* Trajectory comparison: dl_solve against oracle.agd on the same seeded instance, with and without
  Jacobi preconditioning and gamma continuation.  The library hands the gradient fp32 duals
  (R7); the oracle's AGD evaluates at fp64 D lam2 (the paper's AGD), so this comparison uses the
  oracle's test-harness option mu_fp32=True to follow the same points; the remaining
  differences are reduction orders (fp64).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from oracle.agd import AgdConfig, agd  # noqa: E402
from oracle.dual import Problem, apply_A, dual_eval  # noqa: E402
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


@pytest.mark.parametrize("cfg", [AgdConfig(gamma0=0.01, mu_fp32=True), AgdConfig(gamma0=0.01, jacobi=False, mu_fp32=True),
                                 AgdConfig(gamma0=0.16, gamma_min=0.01, halve_every=25, mu_fp32=True)])
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
    h, _, tr = run_both(inst, 3, AgdConfig(gamma0=0.05, max_step=1e-2, mu_fp32=True))
    np.testing.assert_allclose(h["g"], tr.g, rtol=1e-10)
    np.testing.assert_allclose(h["eta"], tr.eta, rtol=1e-10)
    np.testing.assert_allclose(h["gnorm"], tr.gnorm, rtol=1e-9)
    np.testing.assert_allclose(h["infeas"], tr.infeas, rtol=1e-9)


def test_solve_converges_like_oracle():
    """Reaching a 1e-3 relative dual gap takes the same number of iterations (+-2%)."""
    inst = generate(GenConfig(num_sources=300, num_dests=20, nnz_per_source=5, seed=11))
    cfg = AgdConfig(gamma0=0.01)  # the paper's fp64 AGD: iterations-to-gap must still agree
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
    cfg = AgdConfig(gamma0=0.01, mu_fp32=True)
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


def _iterate_pin(inst, iters, kind=0, r=1.0, u=1.0, gamma0=0.16, gamma_min=0.01, every=1):
    """Step the solver through the C ABI; at every `every`-th iterate compare the accumulated
    A x*(mu_t) - b and g(mu_t) with the fp64 oracle at the same mu_t (R12 tolerance)."""
    from paper_2603_04621_b200 import _lib as L
    gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=u)
    gp.set_jacobi(gp.row_sqnorms())
    gp.agd_init(gamma0=gamma0, gamma_min=gamma_min, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
    P = Problem.from_instance(inst, kind=kind, r=r, u=(np.inf if kind == 0 else u))
    grad_d, obj_d = gp.new_grad_buffers()
    checked = 0
    for t in range(iters):
        mu = gp.point().astype(np.float64)           # the point the next evaluation uses
        L.dl_agd_eval(gp.h)
        if t % every == 0:
            L.dl_agd_gradient(gp.h, grad_d, obj_d)
            gp.sync()
            grad, obj = grad_d.cpu().numpy(), obj_d.cpu().numpy()
            ev = dual_eval(P, mu, _gamma_t(t, gamma0, gamma_min))
            absAx = apply_A(P, np.abs(ev.x))
            err = np.abs(grad - ev.grad)
            tol = 1e-5 * (absAx + np.abs(P.b)) + 1e-12
            assert np.all(err <= tol), (t, float(np.max(err / tol)))
            gscale = float(np.abs(P.c) @ np.abs(ev.x)) + abs(ev.reg) + float(np.abs(mu) @ (absAx + np.abs(P.b)))
            assert abs(obj[0] - ev.g) <= 1e-5 * gscale + 1e-12, (t, obj[0], ev.g)
            checked += 1
        L.dl_dual_step(gp.h)
    hist = gp.history()
    gp.close()
    return checked, hist


def _gamma_t(t, gamma0, gamma_min):
    return max(gamma0 * 0.5 ** (t // 25), gamma_min) if gamma_min else gamma0


@pytest.mark.parametrize("name,kind,r,u", [("tiny", 0, 1.0, 1.0), ("mid_simplex", 0, 1.0, 1.0),
                                            ("mid_boxcut", 1, 3.0, 1.0), ("bigJ_hot", 0, 1.0, 1.0)])
def test_every_iterate_matches_oracle_at_the_visited_point(name, kind, r, u):
    """The GPU solver's whole trajectory, pinned iterate by iterate to the paper's fp64 dual at
    the points it actually visits (no oracle precision option involved)."""
    cfgs = {"tiny": CONFIGS["tiny"],
            "mid_simplex": GenConfig(num_sources=4000, num_dests=300, nnz_per_source=60, seed=50),
            "mid_boxcut": GenConfig(num_sources=3000, num_dests=300, nnz_per_source=60, num_families=2, seed=51),
            "bigJ_hot": GenConfig(num_sources=3000, num_dests=60000, nnz_per_source=40, seed=52)}
    inst = generate(cfgs[name])
    iters, every = (200, 1) if name == "tiny" else (150, 5)
    checked, hist = _iterate_pin(inst, iters, kind, r, u, every=every)
    assert checked == (iters + every - 1) // every
    assert hist.size == iters
