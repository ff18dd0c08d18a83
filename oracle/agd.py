"""Dual ascent drivers (oracle, float64).

* ``agd`` -- the Maximizer of PAPER.md Table 1: projected
  Nesterov accelerated gradient ascent on g over lambda >= 0 (PAPER.md:92,
  694-706) with a step from a running local Lipschitz estimate capped by
  max-step-size, gamma continuation with the max step scaled
  with gamma, run in Jacobi-preconditioned dual
  coordinates.  The paper does not print the update
  formulas (it cites AcceleratedGradientDescent.scala); the exact formulas are
  DESIGN.md readings R5-R8, written here step by step in that order:

    t = 0, 1, ...:   gamma_t = max(gamma0 * 2^-floor(t/period), gamma_min)
      1  mu_t   = D * lam2                  point handed to the gradient oracle (fp64, the
                                            paper's AGD; ``mu_fp32=True`` is a test-harness option
                                            that rounds it to float32 like a caller handing the
                                            gradient fp32 duals -- never the default)
      2  G_t    = D * (A x*(mu_t) - b)      preconditioned gradient; g_t = g(mu_t)
      3  eta_t  = init_step                                          if t = 0
                = min(eta_{t-1} * gamma_t/gamma_{t-1}, cap(gamma_t))  if gamma changed (R6)
                = min(||lam2 - lam2_prev|| / ||G_t - G_prev||, cap)   otherwise (R5)
         cap(gamma) = max_step * gamma / gamma_ref (gamma_ref = gamma_min, or gamma0 if fixed)
      4  lam1'  = max(lam2 + eta_t G_t, 0)
      5  lam2'  = max(lam1' + (k-1)/(k+2) (lam1' - lam1), 0),  k -> k+1
         (k restarts at 1 whenever gamma changes -- R6)

* ``projected_gradient`` -- lambda <- max(lambda + grad g / L, 0), the plain
  ascent step used in the proof of Appendix A.2.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .dual import Problem, dual_eval, jacobi_diag, row_sqnorms


@dataclasses.dataclass(frozen=True)
class AgdConfig:
    gamma0: float = 0.01
    gamma_min: float | None = None   # None: fixed gamma
    halve_every: int = 25
    max_step: float = 1e-3
    init_step: float = 1e-5
    jacobi: bool = True
    mu_fp32: bool = False            # harness option only (see module docstring, step 1)


def gamma_at(cfg: AgdConfig, t: int) -> float:
    """Continuation schedule: halve every `halve_every` iterations down to gamma_min."""
    if cfg.gamma_min is None:
        return cfg.gamma0
    return max(cfg.gamma0 * 0.5 ** (t // cfg.halve_every), cfg.gamma_min)


def step_cap(cfg: AgdConfig, gamma: float) -> float:
    """Max step proportional to gamma, equal to max_step at gamma_ref."""
    ref = cfg.gamma0 if cfg.gamma_min is None else cfg.gamma_min
    return cfg.max_step * gamma / ref


@dataclasses.dataclass
class AgdTrace:
    g: list           # g(mu_t), one per iteration
    gamma: list
    eta: list
    gnorm: list       # ||G_t||
    infeas: list      # ||(A x* - b)_+||  (original coordinates, Appendix A.2)
    lam1: np.ndarray  # final iterate (preconditioned coordinates)
    lam2: np.ndarray
    d: np.ndarray     # Jacobi diagonal (ones if off)


def agd(P: Problem, iters: int, cfg: AgdConfig = AgdConfig(), callback=None) -> AgdTrace:
    n = P.num_families * P.num_dests
    d = jacobi_diag(row_sqnorms(P)) if cfg.jacobi else np.ones(n)
    lam1 = np.zeros(n)
    lam2 = np.zeros(n)
    lam2_prev = G_prev = None
    eta = cfg.init_step
    k = 1
    gamma_prev = None
    tr = AgdTrace([], [], [], [], [], lam1, lam2, d)
    for t in range(iters):
        gamma = gamma_at(cfg, t)
        if gamma_prev is not None and gamma != gamma_prev:
            k = 1                                                     # R6: momentum restart
        mu = d * lam2                                                 # 1
        if cfg.mu_fp32:
            mu = mu.astype(np.float32).astype(np.float64)
        ev = dual_eval(P, mu, gamma)
        G = d * ev.grad                                               # 2
        if t == 0:                                                    # 3
            eta = cfg.init_step
        elif gamma != gamma_prev:
            eta = min(eta * gamma / gamma_prev, step_cap(cfg, gamma))
        else:
            dl = float(np.linalg.norm(lam2 - lam2_prev))
            dg = float(np.linalg.norm(G - G_prev))
            eta = min(dl / dg, step_cap(cfg, gamma)) if (dl > 0 and dg > 0) else step_cap(cfg, gamma)
        lam1_new = np.maximum(lam2 + eta * G, 0.0)                    # 4
        beta = (k - 1) / (k + 2)
        lam2_new = np.maximum(lam1_new + beta * (lam1_new - lam1), 0.0)  # 5
        tr.g.append(ev.g); tr.gamma.append(gamma); tr.eta.append(eta)
        tr.gnorm.append(float(np.linalg.norm(G)))
        tr.infeas.append(float(np.linalg.norm(np.maximum(ev.grad, 0.0))))
        if callback is not None:
            callback(t, mu, ev)
        lam2_prev, G_prev = lam2, G
        lam1, lam2 = lam1_new, lam2_new
        k += 1
        gamma_prev = gamma
    tr.lam1, tr.lam2 = lam1, lam2
    return tr


def projected_gradient(P: Problem, lam0, gamma, L, iters):
    """lambda_{t+1} = Pi_{R+}(lambda_t + grad g(lambda_t)/L); returns the g sequence."""
    lam = np.asarray(lam0, dtype=np.float64).copy()
    gs = []
    for _ in range(iters):
        ev = dual_eval(P, lam, gamma)
        gs.append(ev.g)
        lam = np.maximum(lam + ev.grad / L, 0.0)
    return gs, lam


__all__ = ["AgdConfig", "AgdTrace", "agd", "gamma_at", "step_cap", "projected_gradient"]
