"""Pins for oracle.dual: dense expansion, finite differences, Danskin minimality,
weak/strong duality against exact LP/QP optima, Lipschitz bound, Jacobi
preconditioning (Lemma 1) and primal scaling.
"""
import dataclasses

import numpy as np
import pytest
from scipy.optimize import linprog, minimize

from oracle.dual import (BOX, BOXCUT, SIMPLEX, Problem, apply_A, dual_eval, expand_dense, jacobi_diag,
                         lagrangian, primal, reduced_costs, row_normalise, row_sqnorms)
from oracle.projection import project
from tests.helpers import lp_constraints, random_feasible_x, tiny_problem

KINDS = [(SIMPLEX, 1.0, np.inf), (BOXCUT, 2.0, 0.7), (BOX, 1.0, 1.0)]


def test_matvecs_match_dense_expansion():
    rng = np.random.default_rng(0)
    for seed in range(40):
        m = 1 + seed % 3
        P = tiny_problem(seed, I=int(rng.integers(1, 9)), J=int(rng.integers(1, 7)), m=m, nu=2.5)
        A = expand_dense(P)
        I, J = P.num_sources, P.num_dests
        x = rng.normal(size=P.nnz)
        xd = np.zeros(I * J)
        for i in range(I):
            for e in range(P.row_ptr[i], P.row_ptr[i + 1]):
                xd[i * J + P.dest[e]] = x[e]
        np.testing.assert_allclose(apply_A(P, x), A @ xd, atol=1e-12)
        lam = rng.normal(size=m * J)
        atl = A.T @ lam
        got = reduced_costs(P, lam) - P.c
        want = np.array([atl[i * J + P.dest[e]] for i in range(I) for e in range(P.row_ptr[i], P.row_ptr[i + 1])])
        np.testing.assert_allclose(got, want, atol=1e-12)
        # adjoint identity <A x, lam> = <x, A^T lam>
        assert abs(np.dot(apply_A(P, x), lam) - np.dot(x, got)) <= 1e-10 * (1 + abs(np.dot(x, got)))


def test_closed_form_1x1():
    """I=J=m=1, a=2, b=1, c=-1, box[0,1], gamma=1 (hand evaluation of Eq. 2)."""
    P = Problem(1, 1, 1, np.array([0, 1]), np.array([0]), np.array([[2.0]]), np.array([-1.0]),
                np.array([1.0]), BOX, 1.0, 1.0)
    ev = dual_eval(P, np.array([0.0]), 1.0)      # y = 1 -> x = 1; grad = 2-1; g = -1 + 1/2
    assert ev.x[0] == 1.0 and ev.grad[0] == 1.0 and ev.g == -0.5
    ev = dual_eval(P, np.array([1.0]), 1.0)      # y = -(2-1) = -1 -> x = 0; g = 0 + 0 + 1*(0-1)
    assert ev.x[0] == 0.0 and ev.grad[0] == -1.0 and ev.g == -1.0
    # inner minimisation by grid over [0,1] agrees
    xs = np.linspace(0, 1, 100001)
    for lam in (0.0, 0.3, 1.0):
        L = -xs + 0.5 * xs ** 2 + lam * (2 * xs - 1)
        assert abs(L.min() - dual_eval(P, np.array([lam]), 1.0).g) < 1e-9


@pytest.mark.parametrize("kind,r,u", KINDS)
def test_finite_difference_gradient(kind, r, u):
    rng = np.random.default_rng(1)
    for seed in range(12):
        P = tiny_problem(seed, I=10, J=6, m=1 + seed % 2, nu=3.0, kind=kind, r=r, u=u)
        gamma = float(rng.choice([0.05, 0.3, 1.0]))
        lam = rng.uniform(0, 2, P.num_families * P.num_dests)
        ev = dual_eval(P, lam, gamma)
        h = 1e-6
        for rr in range(lam.size):
            e = np.zeros(lam.size); e[rr] = h
            fd = (dual_eval(P, lam + e, gamma).g - dual_eval(P, lam - e, gamma).g) / (2 * h)
            assert abs(fd - ev.grad[rr]) <= 1e-5 * (1 + abs(ev.grad[rr])), (rr, fd, ev.grad[rr])


@pytest.mark.parametrize("kind,r,u", KINDS)
def test_danskin_minimality(kind, r, u):
    """g(lambda) = L(x*, lambda) <= L(x, lambda) for every feasible x."""
    rng = np.random.default_rng(2)
    for seed in range(8):
        P = tiny_problem(seed + 50, I=12, J=5, m=2, nu=3.0, kind=kind, r=r, u=u)
        lam = rng.uniform(0, 1.5, 2 * P.num_dests)
        gamma = 0.2
        ev = dual_eval(P, lam, gamma)
        assert abs(lagrangian(P, ev.x, lam, gamma) - ev.g) < 1e-10 * (1 + abs(ev.g))
        for _ in range(100):
            x = random_feasible_x(P, rng)
            assert lagrangian(P, x, lam, gamma) >= ev.g - 1e-9


@pytest.mark.parametrize("kind,r,u", KINDS[:2])
def test_weak_duality_vs_exact_lp(kind, r, u):
    """g_gamma(lambda) <= c^T x_LP + gamma/2 ||x_LP||^2 for every lambda >= 0 (HiGHS optimum)."""
    rng = np.random.default_rng(3)
    for seed in range(6):
        P = tiny_problem(seed + 100, I=15, J=6, m=1 + seed % 2, nu=3.0, kind=kind, r=r, u=u)
        Aub, bub, bounds = lp_constraints(P)
        res = linprog(P.c, A_ub=Aub, b_ub=bub, bounds=bounds, method="highs")
        assert res.status == 0
        xlp = res.x
        for gamma in (0.01, 0.1, 1.0):
            ub = float(P.c @ xlp) + 0.5 * gamma * float(xlp @ xlp)
            for _ in range(30):
                lam = rng.exponential(rng.choice([0.1, 1.0, 10.0]), P.num_families * P.num_dests)
                assert dual_eval(P, lam, gamma).g <= ub + 1e-9


def _qp_optimum(P: Problem, gamma):
    """p_gamma* = min_{x in C, Ax<=b} c^T x + gamma/2 ||x||^2 by SLSQP on the dense form."""
    Aub, bub, bounds = lp_constraints(P)
    f = lambda x: P.c @ x + 0.5 * gamma * x @ x
    jac = lambda x: P.c + gamma * x
    cons = {"type": "ineq", "fun": lambda x: bub - Aub @ x, "jac": lambda x: -Aub}
    res = minimize(f, np.zeros(P.nnz), jac=jac, bounds=bounds, constraints=[cons], method="SLSQP",
                   options={"ftol": 1e-13, "maxiter": 2000})
    assert res.success, res.message
    return res.fun


def _dual_max(P: Problem, gamma, iters=6000):
    """max g by projected gradient ascent with step 1/L, L = sigma_max(A)^2/gamma."""
    A = expand_dense(P)
    L = np.linalg.norm(A, 2) ** 2 / gamma
    lam = np.zeros(A.shape[0])
    best = -np.inf
    for _ in range(iters):
        ev = dual_eval(P, lam, gamma)
        best = max(best, ev.g)
        lam = np.maximum(lam + ev.grad / L, 0)
    return best, lam


def test_strong_duality_smoothed():
    """max_lambda g_gamma = p_gamma* ('by strong duality')."""
    for seed in range(3):
        P = tiny_problem(seed + 200, I=6, J=4, m=1, nu=2.5)
        gamma = 0.5
        gmax, _ = _dual_max(P, gamma, iters=40000)
        p = _qp_optimum(P, gamma)
        assert abs(gmax - p) <= 1e-6 * (1 + abs(p)), (gmax, p)


def test_lp_recovery_small_gamma():
    """As gamma -> 0 the smoothed optimum (= max g_gamma, test above) approaches the LP
    optimum: lp <= p_gamma* <= lp + gamma/2 max_{x in C}||x||^2 (Lemma 2 of ECLIPSE)."""
    P = tiny_problem(300, I=6, J=4, m=1, nu=2.5)
    Aub, bub, bounds = lp_constraints(P)
    lp = linprog(P.c, A_ub=Aub, b_ub=bub, bounds=bounds, method="highs").fun
    for gamma in (0.05, 0.01, 0.001):
        gmax = _qp_optimum(P, gamma)
        bound = 0.5 * gamma * P.num_sources * P.r ** 2       # ||x||^2 <= sum_i r^2 on the simplex
        assert lp - 1e-6 <= gmax + 1e-9 and gmax <= lp + bound + 1e-6


def test_gradient_lipschitz():
    rng = np.random.default_rng(5)
    for seed in range(10):
        P = tiny_problem(seed + 400, I=10, J=5, m=2, nu=3.0)
        A = expand_dense(P)
        gamma = 0.3
        L = np.linalg.norm(A, 2) ** 2 / gamma
        for _ in range(20):
            l1, l2 = rng.uniform(0, 2, A.shape[0]), rng.uniform(0, 2, A.shape[0])
            d = np.linalg.norm(dual_eval(P, l1, gamma).grad - dual_eval(P, l2, gamma).grad)
            assert d <= L * np.linalg.norm(l1 - l2) * (1 + 1e-9)


def test_jacobi_row_normalisation():
    rng = np.random.default_rng(6)
    for seed in range(10):
        P = tiny_problem(seed + 500, I=12, J=6, m=2, nu=3.0)
        P2, d = row_normalise(P)
        A, A2 = expand_dense(P), expand_dense(P2)
        norms = np.linalg.norm(A2, axis=1)
        nz = np.linalg.norm(A, axis=1) > 0
        np.testing.assert_allclose(norms[nz], 1.0, atol=1e-12)
        np.testing.assert_array_equal(d[~nz], 1.0)                       # zero rows left unscaled
        np.testing.assert_allclose(d[nz] ** 2, 1.0 / np.diag(A @ A.T)[nz], rtol=1e-12)
        for _ in range(200):                                              # feasible set preserved
            x = rng.uniform(0, 1, P.nnz)
            assert np.all(apply_A(P, x) <= P.b) == np.all(apply_A(P2, x) <= P2.b)


def test_jacobi_as_dual_change_of_variables():
    """g'(lam') = g(D lam') and grad g'(lam') = D grad g(D lam'): preconditioning the
    rows equals evaluating the original dual at D lam' (how the CUDA path applies D)."""
    rng = np.random.default_rng(7)
    for seed in range(10):
        P = tiny_problem(seed + 600, I=12, J=6, m=1 + seed % 2, nu=3.0)
        P2, d = row_normalise(P)
        lamp = rng.uniform(0, 3, d.size)
        e2 = dual_eval(P2, lamp, 0.1)
        e1 = dual_eval(P, d * lamp, 0.1)
        assert abs(e2.g - e1.g) <= 1e-12 * (1 + abs(e1.g))
        np.testing.assert_allclose(e2.grad, d * e1.grad, atol=1e-12)
        assert np.allclose(e2.x, e1.x, atol=1e-12)


def test_lemma1_gershgorin():
    """Lemma 1: i.i.d. user blocks, D_exp from E||A_r||^2 ->
    diag(E[~A ~A^T]) = I and kappa <= (1+(m-1)eta)/(1-(m-1)eta)."""
    rng = np.random.default_rng(8)
    J = 1
    for m, rho in ((2, 0.1), (3, 0.05), (2, 0.3)):
        cov = np.full((m, m), rho) + (1 - rho) * np.eye(m)
        scales = np.array([1.0, 4.0, 0.3][:m])
        Lc = np.linalg.cholesky(cov)
        I, trials = 400, 300
        M = np.zeros((m, m))
        for _ in range(trials):           # each block A_i is diag over one destination: m x 1 column
            z = (Lc @ rng.normal(size=(m, I))) * scales[:, None]
            M += z @ z.T
        M /= trials                        # estimate of E[A A^T]
        Dexp = np.diag(1 / np.sqrt(np.diag(M)))
        Mt = Dexp @ M @ Dexp
        np.testing.assert_allclose(np.diag(Mt), 1.0, atol=1e-12)
        eta = np.max(np.abs(Mt - np.diag(np.diag(Mt))))
        assert (m - 1) * eta < 1
        ev = np.linalg.eigvalsh(Mt)
        kappa = ev[-1] / ev[0]
        assert kappa <= (1 + (m - 1) * eta) / (1 - (m - 1) * eta) * (1 + 1e-12)


def test_primal_scaling_two_views():
    """View (i) gamma_i = gamma v_i^2 on x equals view (ii): z = v x with c' = c/v,
    A' = A/v and z in v C, solved with the unscaled projection."""
    rng = np.random.default_rng(9)
    for seed in range(10):
        for kind, r, u in KINDS:
            base = tiny_problem(seed + 700, I=10, J=5, m=1 + seed % 2, nu=3.0, kind=kind, r=r, u=u)
            v = rng.uniform(0.3, 3.0, base.num_sources)
            P = dataclasses.replace(base, v=v)
            lam = rng.uniform(0, 2, P.num_families * P.num_dests)
            gamma = 0.2
            x = primal(P, lam, gamma)
            s = reduced_costs(base, lam)
            for i in range(P.num_sources):
                sl = P.block(i)
                if sl.stop == sl.start:
                    continue
                z = project(kind, -(s[sl] / v[i]) / gamma, r * v[i], u * v[i])
                np.testing.assert_allclose(z / v[i], x[sl], atol=1e-12)
            # and the objective terms agree: gamma/2 ||z||^2 = gamma/2 sum v_i^2 ||x_i||^2
            ev = dual_eval(P, lam, gamma)
            zz = sum((v[i] ** 2) * np.sum(x[P.block(i)] ** 2) for i in range(P.num_sources))
            assert abs(ev.reg - 0.5 * gamma * zz) < 1e-12 * (1 + zz)


def test_empty_blocks_and_zero_rows():
    P = Problem(3, 3, 1, np.array([0, 2, 2, 3]), np.array([0, 1, 1]), np.array([[1.0, 2.0, 0.5]]),
                np.array([-1.0, -2.0, -0.5]), np.array([0.5, 0.5, 1.0]))
    ev = dual_eval(P, np.zeros(3), 0.5)
    assert ev.grad[2] == -1.0                      # destination 2 has no edges: grad = -b
    assert row_sqnorms(P)[2] == 0 and jacobi_diag(row_sqnorms(P))[2] == 1.0
