"""Euclidean projections onto the per-block simple-constraint polytopes (oracle).

PAPER.md:125-134 (Sec. 3.2, "per-user capacity" Eq. 4 and "feasibility" Eq. 5,
and "Simple constraints": "box-cut" or "simplex" inequality constraints applied
to each block independently).  Polytopes, with r > 0 the sum cap and u > 0 the
per-coordinate cap:

    simplex(r)     = {x : x >= 0, sum x <= r}
    boxcut(u, r)   = {x : 0 <= x <= u, sum x <= r}
    box(u)         = {x : 0 <= x <= u}

All in float64; written for clarity, not speed.
"""
from __future__ import annotations

import numpy as np

SIMPLEX, BOXCUT, BOX = 0, 1, 2


def project_box(y, u):
    """Coordinatewise clamp to [0, u]: the projection onto box(u)."""
    return np.clip(np.asarray(y, dtype=np.float64), 0.0, u)


def project_simplex(y, r):
    """Projection onto simplex(r) = {x >= 0, sum x <= r}.

    Inequality form: if the nonnegative clamp already satisfies the cap it is
    the projection; otherwise the projection lies on the face sum x = r and is
    max(y - theta, 0) with theta from the sorted prefix sums (the classical
    sort-and-threshold rule: rho = max{k : mu_k - (sum_{i<=k} mu_i - r)/k > 0}).
    """
    y = np.asarray(y, dtype=np.float64)
    if y.size == 0:
        return y.copy()
    x0 = np.maximum(y, 0.0)
    if x0.sum() <= r:
        return x0
    mu = np.sort(y)[::-1]
    cs = np.cumsum(mu)
    k = np.arange(1, y.size + 1)
    ok = mu - (cs - r) / k > 0
    rho = int(k[ok][-1])
    theta = (cs[rho - 1] - r) / rho
    return np.maximum(y - theta, 0.0)


def _capped_sum(y, u, theta):
    return float(np.clip(y - theta, 0.0, u).sum())


def project_boxcut(y, u, r):
    """Projection onto boxcut(u, r) = {0 <= x <= u, sum x <= r}.

    KKT: x = clip(y - theta, 0, u) with theta >= 0 and theta * (r - sum x) = 0.
    h(theta) = sum clip(y - theta, 0, u) is continuous, nonincreasing and linear
    between the breakpoints {y_j} U {y_j - u}; if h(0) <= r then theta = 0,
    otherwise theta is found by evaluating h at every breakpoint and linearly
    interpolating inside the bracketing segment.
    """
    y = np.asarray(y, dtype=np.float64)
    if y.size == 0:
        return y.copy()
    if _capped_sum(y, u, 0.0) <= r:
        return np.clip(y, 0.0, u)
    bps = np.unique(np.concatenate([[0.0], y, y - u]))
    bps = bps[bps >= 0.0]
    h = np.array([_capped_sum(y, u, t) for t in bps])
    # h(bps[0]=0) > r >= h(max y) = 0: find the first breakpoint with h <= r
    i = int(np.flatnonzero(h <= r)[0])
    t1, t2, h1, h2 = bps[i - 1], bps[i], h[i - 1], h[i]
    theta = t1 + (h1 - r) * (t2 - t1) / (h1 - h2)
    return np.clip(y - theta, 0.0, u)


def project(kind, y, r, u):
    if kind == SIMPLEX:
        return project_simplex(y, r)
    if kind == BOXCUT:
        return project_boxcut(y, u, r)
    if kind == BOX:
        return project_box(y, u)
    raise ValueError(kind)
