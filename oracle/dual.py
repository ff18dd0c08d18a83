"""Ridge-regularised dual of the matching LP (oracle, float64).

PAPER.md:75-91 (Sec. 3.1): LP  min c^T x  s.t.  A x <= b, x in C; dual

    g(lambda) = min_{x in C} c^T x + (gamma/2)||x||^2 + lambda^T (A x - b)

with, by Danskin, grad g(lambda) = A x*_gamma(lambda) - b and
x*_gamma(lambda) = Pi_C(-(A^T lambda + c)/gamma).

Matching structure (Definition 1): A = [D_{k i}] with every
D_{k i} diagonal, so (A^T lambda)_{(i,j)} = sum_k a_{k i j} lambda_{k j} and
(A x)_{k j} = sum_i a_{k i j} x_{i j}; C is a product of per-source polytopes,
so Pi_C is a per-source projection.

Primal scaling, perspective (i): the regulariser becomes
(gamma/2) x^T D_v^2 x.  With v constant on each source block (reading R4 of
DESIGN.md) block i sees gamma_i = gamma v_i^2 and
x*_i = Pi_{C_i}(-s_i / gamma_i), s_ij = c_ij + sum_k a_kij lambda_kj.

Jacobi row normalisation: D_rr = 1/||A_r*||_2 (rows with
zero norm keep D_rr = 1); A' = D A, b' = D b.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .projection import BOX, BOXCUT, SIMPLEX, project


@dataclasses.dataclass
class Problem:
    """float64 view of one matching LP (or one shard of it)."""
    num_sources: int
    num_dests: int
    num_families: int
    row_ptr: np.ndarray        # int64 [I+1]
    dest: np.ndarray           # int64 [nnz]
    a: np.ndarray              # float64 [m, nnz]
    c: np.ndarray              # float64 [nnz]
    b: np.ndarray              # float64 [m*J]
    kind: int = SIMPLEX
    r: float = 1.0             # sum cap
    u: float = np.inf          # coordinate cap (box-cut / box)
    v: np.ndarray | None = None  # per-source primal scale v_i > 0 (None: no scaling)

    @staticmethod
    def from_instance(inst, kind=SIMPLEX, r=1.0, u=np.inf, v=None) -> "Problem":
        return Problem(inst.num_sources, inst.num_dests, inst.num_families,
                       np.asarray(inst.row_ptr, dtype=np.int64),
                       np.asarray(inst.dest, dtype=np.int64),
                       np.asarray(inst.a, dtype=np.float64).reshape(inst.num_families, -1),
                       np.asarray(inst.c, dtype=np.float64),
                       np.asarray(inst.b, dtype=np.float64),
                       kind, float(r), float(u),
                       None if v is None else np.asarray(v, dtype=np.float64))

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def block(self, i):
        return slice(int(self.row_ptr[i]), int(self.row_ptr[i + 1]))

    def gamma_i(self, gamma, i):
        return gamma if self.v is None else gamma * self.v[i] ** 2


def reduced_costs(P: Problem, lam) -> np.ndarray:
    """s_e = c_e + (A^T lambda)_e = c_ij + sum_k a_kij lambda_kj."""
    lam = np.asarray(lam, dtype=np.float64)
    J = P.num_dests
    s = P.c.copy()
    for k in range(P.num_families):
        s += P.a[k] * lam[k * J + P.dest]
    return s


def primal(P: Problem, lam, gamma) -> np.ndarray:
    """x*_gamma(lambda) = Pi_C(-(A^T lambda + c)/gamma), block by block."""
    s = reduced_costs(P, lam)
    x = np.zeros(P.nnz)
    for i in range(P.num_sources):
        sl = P.block(i)
        if sl.stop > sl.start:
            x[sl] = project(P.kind, -s[sl] / P.gamma_i(gamma, i), P.r, P.u)
    return x


def apply_A(P: Problem, x) -> np.ndarray:
    """(A x)_{k j} = sum over edges (i, j) of a_kij x_ij  (Definition 1)."""
    J = P.num_dests
    out = np.zeros(P.num_families * J)
    for k in range(P.num_families):
        out[k * J:(k + 1) * J] = np.bincount(P.dest, weights=P.a[k] * x, minlength=J)
    return out


def regulariser(P: Problem, x, gamma) -> float:
    """(gamma/2) x^T D_v^2 x."""
    if P.v is None:
        return 0.5 * gamma * float(np.dot(x, x))
    lens = np.diff(P.row_ptr)
    w = np.repeat(P.v ** 2, lens)
    return 0.5 * gamma * float(np.dot(w * x, x))


@dataclasses.dataclass
class DualEval:
    grad: np.ndarray   # A x* - b   (length m*J)
    g: float           # g(lambda)
    cx: float          # c^T x*
    reg: float         # (gamma/2)||x*||^2_{D_v^2}
    x: np.ndarray      # x*_gamma(lambda)
    Ax: np.ndarray


def dual_eval(P: Problem, lam, gamma) -> DualEval:
    """g(lambda) and grad g(lambda) = A x*(lambda) - b (Eq. 2 and Danskin)."""
    lam = np.asarray(lam, dtype=np.float64)
    x = primal(P, lam, gamma)
    Ax = apply_A(P, x)
    grad = Ax - P.b
    cx = float(np.dot(P.c, x))
    reg = regulariser(P, x, gamma)
    g = cx + reg + float(np.dot(lam, grad))
    return DualEval(grad, g, cx, reg, x, Ax)


def lagrangian(P: Problem, x, lam, gamma) -> float:
    """c^T x + (gamma/2)||x||^2 + lambda^T (A x - b): the function minimised in Eq. 2."""
    return float(np.dot(P.c, x)) + regulariser(P, x, gamma) + float(np.dot(lam, apply_A(P, x) - P.b))


def row_sqnorms(P: Problem) -> np.ndarray:
    """||A_{r*}||_2^2 for every complex row r = k*J + j."""
    J = P.num_dests
    out = np.zeros(P.num_families * J)
    for k in range(P.num_families):
        out[k * J:(k + 1) * J] = np.bincount(P.dest, weights=P.a[k] ** 2, minlength=J)
    return out


def jacobi_diag(row_sq: np.ndarray) -> np.ndarray:
    """D = diag(||A_r*||^-1), D_rr = 1 on zero rows."""
    d = np.ones_like(row_sq)
    nz = row_sq > 0
    d[nz] = 1.0 / np.sqrt(row_sq[nz])
    return d


def row_normalise(P: Problem):
    """(A', b') = (D A, D b) as an explicit new Problem, plus D."""
    d = jacobi_diag(row_sqnorms(P))
    J = P.num_dests
    a2 = np.empty_like(P.a)
    for k in range(P.num_families):
        a2[k] = P.a[k] * d[k * J + P.dest]
    return dataclasses.replace(P, a=a2, b=P.b * d), d


def expand_dense(P: Problem) -> np.ndarray:
    """The (mJ) x (IJ) dense A of Definition 1 (tiny instances only)."""
    I, J, m = P.num_sources, P.num_dests, P.num_families
    if m * J * I * J > 4_000_000:
        raise ValueError("too large to expand")
    A = np.zeros((m * J, I * J))
    for i in range(I):
        for e in range(P.row_ptr[i], P.row_ptr[i + 1]):
            j = P.dest[e]
            for k in range(m):
                A[k * J + j, i * J + j] = P.a[k, e]
    return A


__all__ = ["Problem", "reduced_costs", "primal", "apply_A", "regulariser", "DualEval", "dual_eval",
           "lagrangian", "row_sqnorms", "jacobi_diag", "row_normalise", "expand_dense",
           "SIMPLEX", "BOXCUT", "BOX"]
