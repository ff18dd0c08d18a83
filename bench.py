#!/usr/bin/env python
"""Benchmark of the dual-gradient hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config NAME]

A step is one iteration of the whole hot path (DESIGN.md §8(a) A3-A5): the fused
dual-gradient pass over every edge of the instance, the gradient all-reduce
(N > 1), and the on-device AGD step.  `value` = edges processed by all ranks per
second of device time (max over ranks), i.e. nnz/s per dual-gradient evaluation.
Extra keys: roofline of the fused kernel, the oracle CPU baseline, end-to-end
throughput through the host-buffer C-ABI entry, and time to a 1e-3 relative dual
gap (R11).

N > 1 (torchrun): weak scaling -- rank r owns sources [r I, (r+1) I) of an
instance with N I sources generated shard-locally (synth, Philox chunks); lambda
is replicated and one NCCL all-reduce of the m J + 4 accumulator runs per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "1M_x_10k"           # BASELINE.json configs[1]: 1M x 10k, ~100 nnz/source, simplex, Jacobi, 1 B200
# workload -> (BASELINE.json configs index, projection kind, r, u, description); kinds as in include/dualip.h
WORKLOADS = {
    "tiny": (0, 0, 1.0, 1.0, "simplex (sum x <= 1)"),
    "1M_x_10k": (1, 0, 1.0, 1.0, "simplex (sum x <= 1)"),
    "100M_x_100k": (2, 0, 1.0, 1.0, "simplex (sum x <= 1)"),
    "multifamily_boxcut": (3, 1, 3.0, 1.0, "box-cut (0 <= x <= 1, sum x <= 3), 2 families (capacity + budget)"),
    "powerlaw": (4, 0, 1.0, 1.0, "simplex (sum x <= 1), power-law block lengths 1..10k"),
    "paper_table_25M": (None, 0, 1.0, 1.0, "simplex (sum x <= 1), the paper's timing-table instance"),
}
# The paper's own numbers, another machine's (context, not the target; BASELINE.json publishes none)
PAPER_CONTEXT = ("PAPER.md:455-476 (table): average time per AGD iteration at 25M sources x 10k destinations, "
                 "sparsity 0.001 (~2.5e8 nnz): PyTorch DuaLip 1 GPU 0.27 s (~9.3e8 nnz/s), Scala/Spark DuaLip "
                 "2.46 s; PAPER.md:18 claims >= 10x over distributed-CPU DuaLip to a fixed gap. GPU model not "
                 "stated in the text. Same-shape run here: bench.py --config paper_table_25M")
GAP_TOL = 1e-3
BURN_ITERS = 2500                # solver iterations before the timed steps (~ the 1e-3 gap point)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-gap", action="store_true", help="skip the time-to-gap measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle CPU baseline")
    return ap.parse_args()


def log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def shard_config(name, world):
    from synth.matching import CONFIGS
    import dataclasses
    base = CONFIGS[name]
    return base, dataclasses.replace(base, num_sources=base.num_sources * world)


# --------------------------------------------------------------------------- oracle arms
def oracle_problem(inst, name):
    from oracle.dual import Problem
    _, kind, r, u, _ = WORKLOADS[name]
    return Problem.from_instance(inst, kind=kind, r=r, u=(np.inf if kind == 0 else u))


def oracle_sample(cfg, name, target_s=15.0, max_sources=200_000):
    """Time oracle.dual_eval on growing prefixes of the workload (same law, same
    seeds) until ~target_s of CPU work; returns (nnz/s, description)."""
    import dataclasses
    from oracle.dual import Problem, dual_eval
    from synth.matching import generate_shard, capacities
    n_src = 2000
    while True:
        inst, load = generate_shard(cfg, 0, n_src, threads=4)
        inst.b = capacities(cfg, load * (cfg.num_sources / max(n_src, 1)))
        P = oracle_problem(inst, name)
        lam = np.full(P.num_families * P.num_dests, 0.0)
        t0 = time.process_time()
        w0 = time.perf_counter()
        dual_eval(P, lam, 0.01)
        dt = time.perf_counter() - w0
        if dt * (target_s / max(dt, 1e-9)) and (dt >= target_s / 4 or n_src >= max_sources):
            break
        n_src = min(max_sources, int(n_src * max(2.0, target_s / 4 / max(dt, 1e-3))))
    reps = max(1, int(target_s / max(dt, 1e-3)))
    w0 = time.perf_counter()
    for _ in range(reps):
        dual_eval(P, lam, 0.01)
    dt = (time.perf_counter() - w0) / reps
    return P.nnz / dt, f"oracle.dual.dual_eval (fp64 numpy, per-block sort projection) on the first {n_src} " \
                       f"sources ({P.nnz} nnz) of {cfg.num_sources}, {reps} reps, {dt:.2f} s/eval"


def run_reference(args):
    """The base contract's reference arm for this tier: the fp64 oracle as it stands, on the host
    cores, each step one dual-gradient evaluation of a bounded prefix of the workload (same law,
    same seeds), the prefix sized so that warm-up + steps take about two minutes."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.dual import dual_eval
    from synth.matching import CONFIGS, capacities, generate_shard
    cfg = CONFIGS[args.config]
    budget_s = 120.0 / max(1, args.steps + args.warmup)

    def prefix(n):
        inst, load = generate_shard(cfg, 0, n, threads=4)
        inst.b = capacities(cfg, load * (cfg.num_sources / n))
        return oracle_problem(inst, args.config)
    n_src = min(500, cfg.num_sources)
    P = prefix(n_src)
    lam = np.zeros(P.num_families * P.num_dests)
    t0 = time.perf_counter()
    dual_eval(P, lam, 0.01)
    per_src = (time.perf_counter() - t0) / n_src
    n_src = int(min(cfg.num_sources, 200_000, max(500, budget_s / max(per_src, 1e-9))))
    P = prefix(n_src)
    lam = np.zeros(P.num_families * P.num_dests)
    for _ in range(args.warmup):
        dual_eval(P, lam, 0.01)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dual_eval(P, lam, 0.01)
    dt = time.perf_counter() - t0
    v = P.nnz * args.steps / dt
    sample = (f"oracle.dual.dual_eval (fp64 numpy, 1 thread) on the first {n_src} sources ({P.nnz} nnz) "
              f"of {args.config}, lambda = 0, gamma = 0.01")
    print(json.dumps({
        "impl": "reference", "metric": "nnz/s per dual-gradient eval", "value": v, "unit": "nnz/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "sample": sample},
        "cpu_baseline": {"value": v, "unit": "nnz/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                try:
                    rows.append((float(f[0]), float(f[1]), f[2:6], float(f[6])))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [r for r in rows if r[3] > 50] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(loaded)}


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2603_04621_b200 import MatchingProblem
    from paper_2603_04621_b200 import _lib as L
    from synth.matching import capacities, generate_shard

    rank, world, local = dist_env()
    assert world == args.gpus or "WORLD_SIZE" not in os.environ, "--gpus must match the torchrun world size"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    base, full = shard_config(args.config, world)
    I = base.num_sources
    threads = max(1, (os.cpu_count() or 8) // world)
    t_gen = time.perf_counter()
    inst, load = generate_shard(full, rank * I, (rank + 1) * I, threads=threads)
    load_t = torch.from_numpy(load).to(dev)
    if world > 1:
        dist.all_reduce(load_t)
    inst.b = capacities(full, load_t.cpu().numpy())
    t_gen = time.perf_counter() - t_gen

    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg_idx, kind, proj_r, proj_u, proj_desc = WORKLOADS[args.config]
    log(f"generated {inst.nnz} nnz in {t_gen:.1f} s")
    t_create = time.perf_counter()
    gp = MatchingProblem.from_instance(inst, kind=kind, r=proj_r, u=proj_u, device=local, stream=stream)
    t_create = time.perf_counter() - t_create
    log(f"created in {t_create:.1f} s: {gp.info}")
    if world > 1:
        gp.comm_init(rank, world)
    rowsq = gp.row_sqnorms()
    gp.allreduce(rowsq)
    gp.set_jacobi(rowsq)
    nnz_local = inst.nnz
    nnz_t = torch.tensor([nnz_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(nnz_t)
    nnz_total = float(nnz_t.item())
    m = inst.num_families
    algo_bytes = nnz_local * (8 + 4 * m)

    # ---- timed region: K hot-path steps (eval -> [all-reduce] -> step), events around each fused launch
    acc_ptr, acc_n = L.dl_agd_accumulator(gp.h)
    gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)

    def one_step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        L.dl_agd_eval(gp.h)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:
            L.dl_comm_allreduce(gp.h, acc_ptr, acc_n)
        L.dl_dual_step(gp.h)

    with ClockSampler(local) as clk:
        # burn-in: the solver runs to iteration BURN_ITERS (the regime of the time-to-gap run,
        # deterministic state; ~1 s of load, clocks steady), then W warm-up steps of the timed loop
        gp.solve(BURN_ITERS)
        for _ in range(args.warmup):
            one_step()
        stream.synchronize()
        if world > 1:
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            one_step(evs[k])
        t1.record(stream)
        stream.synchronize()
        if world > 1:
            dist.barrier()
    ms_total = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in evs]
    ms_t = torch.tensor([ms_total, float(np.mean(kern_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total, kern_avg = float(ms_t[0]), float(ms_t[1])
    value = nnz_total * args.steps / (ms_total / 1e3)

    # ---- end to end through the host-buffer entry (pinned host lambda in, gradient + objective out)
    n = gp.n
    _, l2_now = gp.dual()  # the dual point the timed steps were at
    lam_h = torch.from_numpy(l2_now.astype(np.float32)).pin_memory()
    grad_h = torch.zeros(n, dtype=torch.float64).pin_memory()
    obj_h = torch.zeros(4, dtype=torch.float64).pin_memory()
    grad_d, obj_d = gp.new_grad_buffers()
    lam_d = torch.empty(n, dtype=torch.float32, device=dev)

    def e2e_step():
        if world == 1:
            gp.dual_grad_host(lam_h, 0.01, grad_h, obj_h)
        else:  # same public calls composed: H2D, partial gradient, all-reduce, D2H
            lam_d.copy_(lam_h, non_blocking=True)
            L.dl_dual_grad(gp.h, L.ptr(lam_d), 0.01, L.ptr(grad_d), L.ptr(obj_d), L.DL_GRAD_PARTIAL)
            L.dl_comm_allreduce(gp.h, L.ptr(grad_d), n)
            grad_h.copy_(grad_d, non_blocking=True)
            obj_h.copy_(obj_d, non_blocking=True)
            stream.synchronize()
    for _ in range(3):
        e2e_step()
    if world > 1:
        dist.barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = time.perf_counter() - w0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = nnz_total * args.steps / float(e2e_t.item())

    # ---- time to a 1e-3 relative dual gap (continuation 0.16 -> 0.01, Jacobi; R11)
    gap = None
    if not args.no_gap:
        ref_iters = 8000
        gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5,
                    history_cap=ref_iters)
        gp.solve(ref_iters)
        h = gp.history()
        ghat = float(np.max(h["g"]))
        best = np.maximum.accumulate(h["g"])
        hit = np.flatnonzero(ghat - best <= GAP_TOL * abs(ghat))
        t_star = int(hit[0]) + 1 if hit.size else None
        if t_star is not None:
            gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3,
                        init_step=1e-5, history_cap=ref_iters)
            gp.solve(16)  # graph instantiation outside the timed region
            gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3,
                        init_step=1e-5, history_cap=ref_iters)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            gp.solve(t_star)
            b.record(stream)
            stream.synchronize()
            tg = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tg, op=dist.ReduceOp.MAX)
            gap = {"iterations": t_star, "seconds": float(tg.item()) / 1e3, "rel_gap": GAP_TOL,
                   "g_hat": ghat, "reference_iters": ref_iters,
                   "schedule": "gamma 0.16 -> 0.01 halved every 25, max_step 1e-3 at gamma 0.01, Jacobi"}
        else:
            gap = {"iterations": None, "seconds": None, "rel_gap": GAP_TOL, "reference_iters": ref_iters}

    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except OSError:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "latest_fused_ncu.json")))
            if prof.get("workload") == args.config:
                traffic = prof.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            pass
        achieved = algo_bytes / (kern_avg / 1e3) / 1e9
        cpu = None
        if world == 1 and not args.no_cpu:
            v, sample = oracle_sample(base, args.config)
            cpu = {"value": v, "unit": "nnz/s", "cores": 1, "kind": "oracle", "sample": sample}
        out = {
            "metric": "nnz/s per dual-gradient eval", "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 data, f64 scores/accum",
            "data": "synthetic",
            "config": {"workload": (f"{args.config} (BASELINE configs[{cfg_idx}])" if cfg_idx is not None
                                    else f"{args.config} (PAPER.md:455-476 table instance)"),
                       "num_sources_per_gpu": I,
                       "num_dests": base.num_dests, "families": m, "nnz_total": int(nnz_total),
                       "projection": proj_desc, "jacobi": True,
                       "l2": (f"inputs ({8 + 4 * m} B/nnz, {algo_bytes / 1e9:.2f} GB per GPU) exceed the 126 MB L2; "
                              "no flush needed" if algo_bytes > 4 * 126e6 else
                              f"inputs ({algo_bytes / 1e6:.0f} MB) are L2-resident: not a bench workload"),
                       "parallelism": f"dp{world} (sources sharded, lambda replicated, 1 NCCL all-reduce/step)",
                       "step": "fused dual-gradient pass + all-reduce + on-device AGD step",
                       "timed_from_iteration": BURN_ITERS + args.warmup},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "fused_grad_kernel", "kernel_ms": kern_avg,
                         "algorithmic_bytes_per_launch": algo_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "nnz/s", "h2d_bytes_per_step": 4 * n,
                    "d2h_bytes_per_step": 8 * (n + 4)},
            "gpu_launches": 4 * args.steps,  # per step: fused_grad, deferred, agd_reduce, agd_update kernels
            "clocks": clk.summary(),
            "time_to_gap": gap,
            "paper_context": PAPER_CONTEXT,
            "setup": {"generate_s": t_gen, "tile_cap": gp.info["tile_cap"], "tiles": gp.info["num_tiles"],
                      "lambda_in_smem": bool(gp.info["lambda_in_smem"])},
        }
        print(json.dumps(out), flush=True)
    gp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
