"""Pins for oracle.agd: the paper's gamma schedule, a hand-worked two-step AGD
example, monotone ascent of the smoothed dual under step 1/L and the Appendix
A.2 infeasibility bound, convergence to the exact smoothed optimum (SLSQP),
and the qualitative claims of Figs. 4-5.
"""
import os

import numpy as np
import pytest

from oracle.agd import AgdConfig, agd, gamma_at, projected_gradient, step_cap
from oracle.dual import BOX, Problem, dual_eval, expand_dense
from synth.matching import GenConfig, generate
from tests.helpers import tiny_problem
from tests.test_oracle_dual import _qp_optimum

GOLD = os.path.join(os.path.dirname(__file__), "golden", "gamma_schedule.txt")


def test_gamma_schedule_paper_values():
    """'Decaying gamma from 0.16 to 0.01 (halved every 25 iterations)'."""
    cfg = AgdConfig(gamma0=0.16, gamma_min=0.01, halve_every=25)
    n = 0
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if line:
            t, g = line.split()
            assert gamma_at(cfg, int(t)) == pytest.approx(float(g), rel=1e-15)
            n += 1
    assert n >= 6
    # max step proportional to gamma, equal to max-step-size at the floor
    assert step_cap(cfg, 0.01) == pytest.approx(1e-3)
    assert step_cap(cfg, 0.16) == pytest.approx(1.6e-2)
    assert gamma_at(AgdConfig(gamma0=0.01), 500) == 0.01


def test_two_step_worked_example():
    """1x1 LP, a=2, b=1, c=-1, box [0,1], gamma=1, Jacobi D = 1/|a| = 1/2.
    t=0: mu=0 -> x=1, grad=2*1-1=1, G=D*grad=0.5, eta=init=1e-5,
         lam1 = 5e-6, lam2 = lam1 (k=1: no momentum).
    t=1: mu=2.5e-6 (fp64, the paper's AGD) -> x = 1-2mu, grad = 1-4mu, G = 0.5-2mu;
         L = |G-G0|/|lam2-0| = 2mu/5e-6 ~ 1 -> eta = min(1/L, 1e-3) = 1e-3;
         lam1' = lam2 + 1e-3 G; lam2' = lam1' + (1/4)(lam1' - lam1)."""
    P = Problem(1, 1, 1, np.array([0, 1]), np.array([0]), np.array([[2.0]]), np.array([-1.0]),
                np.array([1.0]), BOX, 1.0, 1.0)
    tr = agd(P, 2, AgdConfig(gamma0=1.0))
    assert tr.eta[0] == 1e-5 and tr.g[0] == -0.5
    mu = 2.5e-6
    G1 = 0.5 - 2 * mu
    assert tr.eta[1] == 1e-3
    lam1_0 = 5e-6
    lam1_1 = lam1_0 + 1e-3 * G1
    lam2_1 = lam1_1 + 0.25 * (lam1_1 - lam1_0)
    assert tr.lam1[0] == pytest.approx(lam1_1, rel=1e-12)
    assert tr.lam2[0] == pytest.approx(lam2_1, rel=1e-12)
    assert tr.g[1] == pytest.approx(-(1 - 2 * mu) + 0.5 * (1 - 2 * mu) ** 2 + mu * (2 * (1 - 2 * mu) - 1), rel=1e-12)


def test_projected_gradient_monotone():
    """Ascent lemma: with step 1/L the smoothed dual never decreases."""
    for seed in range(6):
        P = tiny_problem(seed + 900, I=20, J=6, m=1 + seed % 2, nu=3.0)
        gamma = 0.1
        L = np.linalg.norm(expand_dense(P), 2) ** 2 / gamma
        gs, _ = projected_gradient(P, np.zeros(P.num_families * P.num_dests), gamma, L, 300)
        assert np.all(np.diff(gs) >= -1e-10 * (1 + np.abs(gs[1:])))


def test_appendix_a2_bound_along_agd():
    """||(A x*(lam) - b)_+|| <= sqrt(2 L (g* - g(lam))) at every AGD iterate, with g* the exact
    smoothed optimum (SLSQP primal, = max g by strong duality) and L = ||A||^2/gamma."""
    for seed in range(3):
        P = tiny_problem(seed + 950, I=8, J=4, m=1, nu=2.5)
        gamma = 0.5
        gstar = _qp_optimum(P, gamma)
        L = np.linalg.norm(expand_dense(P), 2) ** 2 / gamma
        checked = []

        def cb(t, mu, ev):
            gap = max(gstar - ev.g, 0.0)
            lhs = np.linalg.norm(np.maximum(ev.grad, 0))
            assert lhs <= np.sqrt(2 * L * gap) + 1e-7, (t, lhs, gap)
            checked.append(t)
        agd(P, 400, AgdConfig(gamma0=gamma, max_step=0.05), callback=cb)
        assert len(checked) == 400


def test_agd_reaches_smoothed_optimum():
    for seed in range(3):
        P = tiny_problem(seed + 980, I=8, J=4, m=1, nu=2.5)
        gamma = 0.5
        gstar = _qp_optimum(P, gamma)
        tr = agd(P, 3000, AgdConfig(gamma0=gamma, max_step=0.05))
        assert max(tr.g) <= gstar + 1e-9
        assert gstar - max(tr.g) <= 1e-6 * (1 + abs(gstar))
        assert np.all(tr.lam1 >= 0) and np.all(tr.lam2 >= 0)


@pytest.fixture(scope="module")
def fig_instance():
    return Problem.from_instance(generate(GenConfig(num_sources=300, num_dests=20, nnz_per_source=5, seed=11),
                                          threads=1))


def _iters_to_gap(tr, ghat, tol=1e-3):
    best = np.maximum.accumulate(np.array(tr.g))
    ok = np.flatnonzero(ghat - best <= tol * abs(ghat))
    return int(ok[0]) if ok.size else 10 ** 9


def test_fig4_fig5_qualitative(fig_instance):
    """Fig. 4: Jacobi preconditioning reaches a 1e-3 dual gap sooner; Fig. 5: gamma
    continuation 0.16 -> 0.01 reaches it sooner than fixed 0.01, final g within 0.5%."""
    P = fig_instance
    iters = 1500
    fixed = agd(P, iters, AgdConfig(gamma0=0.01))
    ghat = max(fixed.g)
    nojac = agd(P, iters, AgdConfig(gamma0=0.01, jacobi=False))
    cont = agd(P, iters, AgdConfig(gamma0=0.16, gamma_min=0.01, halve_every=25))
    n_fixed, n_nojac, n_cont = (_iters_to_gap(t, ghat) for t in (fixed, nojac, cont))
    assert n_fixed < n_nojac, (n_fixed, n_nojac)
    assert n_cont < n_fixed, (n_cont, n_fixed)
    assert abs(max(cont.g[-100:]) - ghat) <= 5e-3 * abs(ghat)
