"""Shared test helpers (no method arithmetic: instance construction only)."""
import numpy as np

from synth.matching import GenConfig, generate
from oracle.dual import Problem, SIMPLEX, BOXCUT, BOX


def tiny_instance(seed=0, I=8, J=5, m=1, nu=3.0, law="poisson"):
    cfg = GenConfig(num_sources=I, num_dests=J, nnz_per_source=nu, num_families=m, seed=seed,
                    length_law=law, max_len=max(1, J))
    return generate(cfg, threads=1)


def tiny_problem(seed=0, I=8, J=5, m=1, nu=3.0, kind=SIMPLEX, r=1.0, u=np.inf, v=None):
    return Problem.from_instance(tiny_instance(seed, I, J, m, nu), kind=kind, r=r, u=u, v=v)


def random_feasible_x(P: Problem, rng):
    """A random point of C (per-block polytope)."""
    x = np.zeros(P.nnz)
    for i in range(P.num_sources):
        sl = P.block(i)
        n = sl.stop - sl.start
        if n == 0:
            continue
        w = rng.exponential(1.0, n) * (rng.random(n) < 0.7)
        if P.kind == BOX:
            x[sl] = rng.uniform(0, P.u, n)
            continue
        tot = rng.uniform(0, P.r)
        if w.sum() > 0:
            w = w / w.sum() * tot
        if P.kind == BOXCUT:
            w = np.minimum(w, P.u)
        x[sl] = w
    return x


def lp_constraints(P: Problem):
    """Dense (A_ub, b_ub, bounds) of min c^T x s.t. A x <= b, x in C (tiny only)."""
    nnz = P.nnz
    J, m = P.num_dests, P.num_families
    rows, rhs = [], []
    for k in range(m):
        for j in range(J):
            row = np.zeros(nnz)
            sel = P.dest == j
            row[sel] = P.a[k][sel]
            rows.append(row)
            rhs.append(P.b[k * J + j])
    if P.kind in (SIMPLEX, BOXCUT):
        for i in range(P.num_sources):
            row = np.zeros(nnz)
            row[P.block(i)] = 1.0
            rows.append(row)
            rhs.append(P.r)
    ub = None if P.kind == SIMPLEX else P.u
    return np.array(rows), np.array(rhs), [(0.0, ub)] * nnz
