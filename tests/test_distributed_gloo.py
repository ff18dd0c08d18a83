"""World-size-2 gloo tests of the multi-GPU decomposition, on CPU.

The sharded path is: balanced contiguous source split (dl_plan_shards, the same host code the
GPU path uses), per-rank partial A x* and objective terms, ONE all-reduce of the m*J + 2
buffer, then the same deterministic AGD step on every rank (so lambda stays replicated
without broadcasts).  Here the per-rank partial is the oracle's (no GPU), the all-reduce is
torch.distributed/gloo, and the checks are: shard partials sum to the full gradient, the
generator's shard-local capacities agree, and a 2-rank AGD run reproduces the 1-process run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.agd import AgdConfig, agd, gamma_at, step_cap
from oracle.dual import Problem, dual_eval, jacobi_diag, row_sqnorms
from synth.matching import GenConfig, capacities, generate, generate_shard

CFG = GenConfig(num_sources=600, num_dests=40, nnz_per_source=6, seed=77, chunk=128)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sub(P: Problem, lo: int, hi: int) -> Problem:
    e0, e1 = int(P.row_ptr[lo]), int(P.row_ptr[hi])
    return Problem(hi - lo, P.num_dests, P.num_families, P.row_ptr[lo:hi + 1] - e0, P.dest[e0:e1],
                   P.a[:, e0:e1], P.c[e0:e1], np.zeros_like(P.b), P.kind, P.r, P.u,
                   None if P.v is None else P.v[lo:hi])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_04621_b200 import _lib as L
    full = generate(CFG, threads=1)
    P = Problem.from_instance(full)
    bounds = L.dl_plan_shards(full.row_ptr, world)          # product host planner
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    # (1) the generator reproduces exactly this shard, and capacities from all-reduced loads
    sh, load = generate_shard(CFG, lo, hi, threads=1)
    np.testing.assert_array_equal(sh.dest, full.dest[full.row_ptr[lo]:full.row_ptr[hi]])
    load_t = torch.from_numpy(load)
    dist.all_reduce(load_t)
    np.testing.assert_allclose(capacities(CFG, load_t.numpy()), full.b, rtol=1e-6)
    # (2) Jacobi row norms: shard partials all-reduced = global norms
    Ps = _sub(P, lo, hi)
    rs = torch.from_numpy(row_sqnorms(Ps))
    dist.all_reduce(rs)
    np.testing.assert_allclose(rs.numpy(), row_sqnorms(P), rtol=1e-12)
    d = jacobi_diag(rs.numpy())
    # (3) replicated AGD with one all-reduce of [A_shard x, c^T x, reg] per iteration
    cfg = AgdConfig(gamma0=0.16, gamma_min=0.01, halve_every=25)
    n = P.num_families * P.num_dests
    lam1 = np.zeros(n); lam2 = np.zeros(n); lam2p = Gp = None; eta = cfg.init_step; k = 1; gprev = None
    gs = []
    for t in range(60):
        gamma = gamma_at(cfg, t)
        if gprev is not None and gamma != gprev:
            k = 1
        mu = d * lam2
        ev = dual_eval(Ps, mu, gamma)                       # partial: b is zero on the shard
        buf = torch.from_numpy(np.concatenate([ev.Ax, [ev.cx, ev.reg]]))
        dist.all_reduce(buf)                                 # the ONE collective of the iteration
        Ax, cx, reg = buf[:n].numpy(), float(buf[n]), float(buf[n + 1])
        grad = Ax - P.b
        gs.append(cx + reg + float(mu @ grad))
        G = d * grad
        if t == 0:
            eta = cfg.init_step
        elif gamma != gprev:
            eta = min(eta * gamma / gprev, step_cap(cfg, gamma))
        else:
            dl, dg = np.linalg.norm(lam2 - lam2p), np.linalg.norm(G - Gp)
            eta = min(dl / dg, step_cap(cfg, gamma)) if dl > 0 and dg > 0 else step_cap(cfg, gamma)
        l1 = np.maximum(lam2 + eta * G, 0)
        l2 = np.maximum(l1 + (k - 1) / (k + 2) * (l1 - lam1), 0)
        lam2p, Gp, lam1, lam2, k, gprev = lam2, G, l1, l2, k + 1, gamma
    # lambda is identical on every rank without any broadcast
    t2 = torch.from_numpy(lam2.copy())
    ref = t2.clone()
    dist.broadcast(ref, 0)
    assert torch.equal(t2, ref)
    out[rank] = gs
    dist.destroy_process_group()


def test_two_rank_decomposition_matches_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    single = agd(Problem.from_instance(generate(CFG, threads=1)), 60,
                 AgdConfig(gamma0=0.16, gamma_min=0.01, halve_every=25))
    for r in range(world):
        np.testing.assert_allclose(out[r], single.g, rtol=1e-9)
    np.testing.assert_array_equal(out[0], out[1])


def test_shard_plan_balances_nnz():
    from paper_2603_04621_b200 import _lib as L
    inst = generate(GenConfig(num_sources=5000, num_dests=100, length_law="powerlaw", max_len=100, seed=3))
    for world in (2, 4, 8):
        b = L.dl_plan_shards(inst.row_ptr, world)
        nnz = np.diff(inst.row_ptr[b])
        assert nnz.sum() == inst.nnz
        assert nnz.max() <= np.ceil(inst.nnz / world) + np.diff(inst.row_ptr).max()
