"""Pins for oracle.projection against brute force, KKT and closed forms.

PAPER.md:125-134 defines the per-block polytopes (simplex Eq. 4-5, box-cut).
A projection is the unique nearest feasible point; the brute-force pin
enumerates every active-set pattern (each coordinate at 0, free, or at the cap;
sum cap active or not), keeps the feasible candidates and takes the nearest --
a definition independent of the sort/breakpoint rules in the oracle.
"""
import itertools
import os

import numpy as np
import pytest

from oracle.projection import BOX, BOXCUT, SIMPLEX, project, project_box, project_boxcut, project_simplex

GOLD = os.path.join(os.path.dirname(__file__), "golden", "projection_examples.txt")


def brute_simplex(y, r):
    n = y.size
    best, bestd = None, np.inf
    for mask in itertools.product([0, 1], repeat=n):
        S = np.array(mask, bool)
        for sum_active in (False, True):
            x = np.zeros(n)
            if sum_active:
                if not S.any():
                    continue
                th = (y[S].sum() - r) / S.sum()
                x[S] = y[S] - th
            else:
                x[S] = y[S]
            if (x >= -1e-12).all() and x.sum() <= r + 1e-12:
                dd = np.sum((x - y) ** 2)
                if dd < bestd - 1e-15:
                    best, bestd = x, dd
    return best


def brute_boxcut(y, u, r):
    n = y.size
    best, bestd = None, np.inf
    for pat in itertools.product([0, 1, 2], repeat=n):   # 0: zero, 1: free, 2: capped
        pat = np.array(pat)
        F, C = pat == 1, pat == 2
        for sum_active in (False, True):
            x = np.zeros(n)
            x[C] = u
            if sum_active:
                if not F.any():
                    continue
                th = (y[F].sum() + u * C.sum() - r) / F.sum()
                x[F] = y[F] - th
            else:
                x[F] = y[F]
            if (x >= -1e-12).all() and (x <= u + 1e-12).all() and x.sum() <= r + 1e-12:
                dd = np.sum((x - y) ** 2)
                if dd < bestd - 1e-15:
                    best, bestd = x, dd
    return best


def test_simplex_matches_bruteforce():
    rng = np.random.default_rng(0)
    for _ in range(1500):
        n = rng.integers(1, 7)
        y = rng.normal(0, 1.5, n) * rng.choice([0.1, 1, 5])
        r = float(rng.choice([0.5, 1.0, 2.0, 3.7]))
        np.testing.assert_allclose(project_simplex(y, r), brute_simplex(y, r), atol=1e-12)


def test_boxcut_matches_bruteforce():
    rng = np.random.default_rng(1)
    for _ in range(600):
        n = rng.integers(1, 6)
        y = rng.normal(0.5, 1.2, n) * rng.choice([0.3, 1, 4])
        u = float(rng.choice([0.3, 1.0, 2.0]))
        r = float(rng.choice([0.5, 1.0, 2.0, 3.0]))
        np.testing.assert_allclose(project_boxcut(y, u, r), brute_boxcut(y, u, r), atol=1e-12)


@pytest.mark.parametrize("kind", [SIMPLEX, BOXCUT])
def test_kkt(kind):
    """x = clip(y - theta, 0, u), theta >= 0, theta (r - sum x) = 0, x feasible."""
    rng = np.random.default_rng(2)
    for _ in range(3000):
        n = rng.integers(1, 65)
        y = rng.normal(0, 2, n)
        r = float(rng.uniform(0.2, 5))
        u = np.inf if kind == SIMPLEX else float(rng.uniform(0.1, 2))
        x = project(kind, y, r, u)
        assert (x >= 0).all() and (x <= u + 1e-12).all() and x.sum() <= r + 1e-9
        free = (x > 1e-12) & (x < u - 1e-12)
        if free.any():
            th = float(np.mean(y[free] - x[free]))
            np.testing.assert_allclose(y[free] - x[free], th, atol=1e-9)
        else:  # theta pinned by the inactive coordinates only: any admissible value
            lo = max([0.0] + list(y[x <= 1e-12]))          # x_j = 0  needs y_j - theta <= 0
            hi = min([np.inf] + list(y[x >= u - 1e-12] - u))  # x_j = u  needs y_j - theta >= u
            assert lo <= hi + 1e-9
            th = lo
        assert th >= -1e-9
        assert abs(th * (r - x.sum())) <= 1e-8 * max(1, abs(th))
        np.testing.assert_allclose(np.clip(y - th, 0, u), x, atol=1e-9)


def test_closed_forms():
    # already feasible: unchanged
    np.testing.assert_allclose(project_simplex(np.array([0.2, 0.3]), 1.0), [0.2, 0.3])
    # all negative: origin
    np.testing.assert_allclose(project_simplex(np.array([-1.0, -2.0]), 1.0), [0.0, 0.0])
    # equal scores split the cap evenly: x_j = r/n
    for n in (1, 3, 17):
        np.testing.assert_allclose(project_simplex(np.full(n, 5.0), 2.0), np.full(n, 2.0 / n))
    # box: componentwise clamp
    np.testing.assert_allclose(project_box(np.array([0.2, 1.4, -0.1]), 1.0), [0.2, 1.0, 0.0])
    # empty block
    assert project_simplex(np.zeros(0), 1.0).size == 0


def test_golden_examples():
    """Hand-derived examples, each line citing its derivation (tests/golden/)."""
    n = 0
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        kind, r, u, ys, xs = [f.strip() for f in line.split("|")]
        y = np.array([float(v) for v in ys.split()])
        x = np.array([float(v) for v in xs.split()])
        k = {"simplex": SIMPLEX, "boxcut": BOXCUT, "box": BOX}[kind]
        np.testing.assert_allclose(project(k, y, float(r), float(u)), x, atol=1e-12)
        n += 1
    assert n >= 6


def test_reductions_between_polytopes():
    rng = np.random.default_rng(3)
    for _ in range(500):
        y = rng.normal(0, 2, rng.integers(1, 20))
        r = float(rng.uniform(0.3, 3))
        # u >= r: the coordinate cap is implied by the sum cap -> simplex
        np.testing.assert_allclose(project_boxcut(y, r * 1.5, r), project_simplex(y, r), atol=1e-12)
        # r >= n u: the sum cap is implied -> box
        u = float(rng.uniform(0.1, 1))
        np.testing.assert_allclose(project_boxcut(y, u, y.size * u + 1), project_box(y, u), atol=1e-12)


@pytest.mark.parametrize("kind", [SIMPLEX, BOXCUT, BOX])
def test_idempotent_nonexpansive(kind):
    rng = np.random.default_rng(4)
    for _ in range(500):
        n = rng.integers(1, 30)
        p, q = rng.normal(0, 2, n), rng.normal(0, 2, n)
        r, u = 1.3, (np.inf if kind == SIMPLEX else 0.7)
        Pp, Pq = project(kind, p, r, u), project(kind, q, r, u)
        np.testing.assert_allclose(project(kind, Pp, r, u), Pp, atol=1e-12)
        assert np.linalg.norm(Pp - Pq) <= np.linalg.norm(p - q) + 1e-12
