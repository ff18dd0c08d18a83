"""Appendix-B synthetic matching LPs, source-chunked so any shard is reproducible.

PAPER.md:673-682 (Appendix B, "Synthetic LP construction"): per resource j a
lognormal breadth normalised to probabilities p_j, K_j ~ Poisson(p_j I nu)
incident requests, and on each edge c_ij = min(v_j u_i eps_ij, c_max),
a_ij = s_j c_ij.  PAPER.md:684-689 ("Source capacities and right-hand side"):
greedy load l_j (each request puts its largest a_ij on that resource),
b_j = rho_j (l_j + eps), rho_j ~ U[0.5, 1]; the value matrix is negated for the
minimisation convention.

Reading (R9): the per-resource Poisson draw is *Poissonised* per
source: with K_j ~ Poisson(p_j I nu) and uniformly chosen requests, request i
meets resource j ~ Poisson(p_j nu) times independently, so a source's degree is
Poisson(nu) and its destinations are i.i.d. Categorical(p) draws (duplicates
merged).  This is the same distribution up to the with/without-replacement
detail and lets every source chunk be drawn from its own counter-keyed Philox
stream, so rank r of N generates exactly its shard of the same instance.

For m > 1 families (BASELINE configs[3], "capacity + budget") family 0 is the
paper's a = s_j c; family k >= 1 is a = s_kj * eps'_ij with fresh lognormal
noise (a family proportional to c would make rows of A parallel, violating the
full-row-rank assumption of PAPER.md:229).
"""
from __future__ import annotations

import dataclasses
import mmap
import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor

import numpy as np

__all__ = ["GenConfig", "Instance", "CONFIGS", "dest_params", "generate_shard", "generate"]


@dataclasses.dataclass(frozen=True)
class GenConfig:
    num_sources: int                 # I
    num_dests: int                   # J
    nnz_per_source: float = 100.0    # nu (mean degree, Poisson law)
    length_law: str = "poisson"      # "poisson" | "powerlaw"
    powerlaw_alpha: float = 2.0      # P(len = n) ~ n^-alpha on [1, max_len]
    max_len: int = 10_000
    num_families: int = 1            # m
    seed: int = 0
    sigma_breadth: float = 1.0
    sigma_value: float = 0.5         # v_j
    sigma_resp: float = 0.5          # u_i
    sigma_noise: float = 0.25        # eps_ij
    sigma_scale: float = 1.0         # s_j
    c_max: float = 10.0
    slack_eps: float = 1e-3
    rho_lo: float = 0.5
    rho_hi: float = 1.0
    chunk: int = 1 << 16             # sources per RNG chunk (fixed: part of the instance identity)


@dataclasses.dataclass
class Instance:
    """Source-major CSR of the matching LP (Definition 1).

    row_ptr[i]..row_ptr[i+1] are source i's eligible edges, dest ascending.
    a[k, e] is diag(D_{k i})_j of edge e=(i,j); c[e] is the (negated) value; b is
    family-major, b[k*J + j].  All float data is float32 (the stored precision).
    """
    num_sources: int
    num_dests: int
    num_families: int
    row_ptr: np.ndarray   # int64 [I+1]
    dest: np.ndarray      # int32 [nnz]
    a: np.ndarray         # float32 [m, nnz]
    c: np.ndarray         # float32 [nnz]
    b: np.ndarray         # float32 [m*J]
    source_offset: int = 0  # global id of local source 0 (shards)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


# BASELINE.json "configs" (index-aligned).  Sizes are the full ones; tests use
# scaled copies with the same structure.
CONFIGS = {
    "tiny": GenConfig(num_sources=1000, num_dests=50, nnz_per_source=10.0, seed=1),
    "1M_x_10k": GenConfig(num_sources=1_000_000, num_dests=10_000, nnz_per_source=100.0, seed=2),
    "100M_x_100k": GenConfig(num_sources=100_000_000, num_dests=100_000, nnz_per_source=50.0, seed=3),
    "multifamily_boxcut": GenConfig(num_sources=10_000_000, num_dests=10_000, nnz_per_source=100.0,
                                    num_families=2, seed=4),
    "powerlaw": GenConfig(num_sources=330_000_000, num_dests=100_000, length_law="powerlaw",
                          powerlaw_alpha=2.0, max_len=10_000, seed=5),
    # the paper's per-iteration timing table: 25M sources x 10k destinations,
    # sparsity 0.001 (10 eligible destinations per source); context, not a BASELINE config
    "paper_table_25M": GenConfig(num_sources=25_000_000, num_dests=10_000, nnz_per_source=10.0, seed=6),
}


def _rng(seed: int, stream: int, index: int) -> np.random.Generator:
    key = np.array([(int(seed) << 8) | int(stream), int(index)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def dest_params(cfg: GenConfig) -> dict:
    """Per-destination draws (Appendix B): p_j, v_j, s_kj, rho_kj."""
    J, m = cfg.num_dests, cfg.num_families
    g = _rng(cfg.seed, 1, 0)
    breadth = g.lognormal(0.0, cfg.sigma_breadth, size=J)
    p = breadth / breadth.sum()
    v = g.lognormal(0.0, cfg.sigma_value, size=J)
    s = g.lognormal(0.0, cfg.sigma_scale, size=(m, J))
    rho = g.uniform(cfg.rho_lo, cfg.rho_hi, size=(m, J))
    cdf = np.cumsum(p)
    cdf[-1] = 1.0
    # guide table for the categorical draw: guide[k] = first j with cdf[j] > k / K (a lower bound of
    # searchsorted(cdf, u, 'right') for u in [k/K, (k+1)/K)); _categorical finishes by stepping up
    K = 1 << max(10, int(np.ceil(np.log2(8 * J))))
    guide = np.searchsorted(cdf, np.arange(K, dtype=np.float64) / K, side="right").astype(np.int64)
    return {"p": p, "cdf": cdf, "guide": guide, "v": v, "s": s, "rho": rho}


def _categorical(dp: dict, u: np.ndarray) -> np.ndarray:
    """searchsorted(cdf, u, side='right'), computed from the guide table (identical result)."""
    cdf, guide = dp["cdf"], dp["guide"]
    K = guide.size
    last = cdf.size - 1
    j = guide[np.minimum((u * K).astype(np.int64), K - 1)]
    np.minimum(j, last, out=j)
    while True:
        step = (cdf[j] <= u) & (j < last)
        if not step.any():
            return j
        j += step


def _powerlaw_cdf(cfg: GenConfig) -> np.ndarray:
    n = np.arange(1, cfg.max_len + 1, dtype=np.float64)
    w = n ** (-cfg.powerlaw_alpha)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return cdf


def _gen_chunk(cfg: GenConfig, dp: dict, chunk_id: int):
    """All sources of one chunk -> (lens, dest, c, a, greedy partial load)."""
    I, J, m = cfg.num_sources, cfg.num_dests, cfg.num_families
    i0 = chunk_id * cfg.chunk
    nsrc = min(cfg.chunk, I - i0)
    g = _rng(cfg.seed, 2, chunk_id)
    if cfg.length_law == "poisson":
        deg = g.poisson(cfg.nnz_per_source, size=nsrc)
    elif cfg.length_law == "powerlaw":
        deg = np.searchsorted(_powerlaw_cdf(cfg), g.random(nsrc), side="right") + 1
    else:
        raise ValueError(cfg.length_law)
    deg = np.minimum(deg, J).astype(np.int64)
    # i.i.d. Categorical(p) draws per source, generated already sorted within
    # each source (uniform order statistics from normalised exponential
    # spacings), so destinations come out ascending without a sort.
    ex = g.standard_exponential(int(deg.sum()) + nsrc)
    cs = np.cumsum(ex)
    ends = np.cumsum(deg + 1) - 1                       # index of each block's (n+1)-th spacing
    starts = ends - deg                                 # first spacing of the block
    base = np.where(starts > 0, cs[np.maximum(starts - 1, 0)], 0.0)
    total = cs[ends] - base
    src = np.repeat(np.arange(nsrc, dtype=np.int64), deg)
    pos = np.arange(src.size, dtype=np.int64) + src     # spacing index of each draw
    u = (cs[pos] - base[src]) / total[src]
    j = _categorical(dp, u)
    np.minimum(j, J - 1, out=j)
    keep = np.ones(src.size, dtype=bool)                # merge duplicate (i, j) draws
    if src.size > 1:
        keep[1:] = (j[1:] != j[:-1]) | (src[1:] != src[:-1])
    src, dest = src[keep], j[keep].astype(np.int32)
    lens = np.bincount(src, minlength=nsrc).astype(np.int64)
    u = g.lognormal(0.0, cfg.sigma_resp, size=nsrc)
    eps = g.lognormal(0.0, cfg.sigma_noise, size=dest.size)
    cval = np.minimum(dp["v"][dest] * u[src] * eps, cfg.c_max)
    a = np.empty((m, dest.size), dtype=np.float32)
    a[0] = (dp["s"][0][dest] * cval).astype(np.float32)
    for k in range(1, m):
        a[k] = (dp["s"][k][dest] * g.lognormal(0.0, cfg.sigma_noise, size=dest.size)).astype(np.float32)
    c = (-cval).astype(np.float32)                      # minimisation convention
    # greedy load: each request adds its largest a_kij (lowest j on ties) to that j
    load = _greedy_load(lens, dest, a, J)
    return lens, dest, c, a, load


_DP_CACHE: dict = {}


_SH: dict = {}  # the shard's output arrays (anonymous shared memory, inherited by forked workers)


def _raw_degrees(cfg: GenConfig, chunk_id: int) -> np.ndarray:
    """The chunk's degree draw (the first draw of its stream, as in _gen_chunk): an upper bound of
    every source's final length (duplicate destinations are merged afterwards)."""
    nsrc = min(cfg.chunk, cfg.num_sources - chunk_id * cfg.chunk)
    g = _rng(cfg.seed, 2, chunk_id)
    if cfg.length_law == "poisson":
        deg = g.poisson(cfg.nnz_per_source, size=nsrc)
    else:
        deg = np.searchsorted(_powerlaw_cdf(cfg), g.random(nsrc), side="right") + 1
    return np.minimum(deg, cfg.num_dests).astype(np.int64)


def _shared(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mmap.mmap(-1, max(n, 1))
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def _shard_job(args):
    """One chunk's slice [lo, hi) written into the shared arrays at edge offset e_raw / source
    offset s_off; returns (edges written, greedy-load partial)."""
    cfg, cid, lo, hi, e_raw, s_off = args
    dp = _DP_CACHE.get(cfg)
    if dp is None:
        dp = _DP_CACHE[cfg] = dest_params(cfg)
    lens, dest, c, a, ld = _gen_chunk(cfg, dp, cid)
    e0, e1 = int(lens[:lo].sum()), int(lens[:hi].sum())
    if lo != 0 or hi != lens.size:  # partial chunk: the greedy load of the kept sources only
        ld = _greedy_load(lens[lo:hi], dest[e0:e1], a[:, e0:e1], cfg.num_dests)
    n = e1 - e0
    _SH["lens"][s_off:s_off + hi - lo] = lens[lo:hi]
    _SH["dest"][e_raw:e_raw + n] = dest[e0:e1]
    _SH["c"][e_raw:e_raw + n] = c[e0:e1]
    _SH["a"][:, e_raw:e_raw + n] = a[:, e0:e1]
    return n, ld


def generate_shard(cfg: GenConfig, src_begin: int, src_end: int, threads: int = 8):
    """Sources [src_begin, src_end) of the instance, plus their greedy-load partial.

    Returns (Instance with b=None, partial_load[m, J] float64).  The full b needs
    the sum of partial loads over all shards (``capacities``).  Chunks are generated by forked
    worker processes straight into shared output arrays sized by the chunks' degree draws (an upper
    bound), then compacted in place: peak memory is about one copy of the shard.
    """
    m, J = cfg.num_families, cfg.num_dests
    c0, c1 = src_begin // cfg.chunk, (max(src_end, src_begin + 1) - 1) // cfg.chunk
    ids = list(range(c0, c1 + 1)) if src_end > src_begin else []
    jobs, e_raw, s_off = [], 0, 0
    for cid in ids:
        i0 = cid * cfg.chunk
        nsrc = min(cfg.chunk, cfg.num_sources - i0)
        lo, hi = max(src_begin, i0) - i0, min(src_end, i0 + nsrc) - i0
        jobs.append((cfg, cid, lo, hi, e_raw, s_off))
        e_raw += int(_raw_degrees(cfg, cid)[lo:hi].sum())
        s_off += hi - lo
    _SH["lens"] = _shared((s_off,), np.int64)
    _SH["dest"] = _shared((e_raw,), np.int32)
    _SH["c"] = _shared((e_raw,), np.float32)
    _SH["a"] = _shared((m, e_raw), np.float32)
    if threads > 1 and len(ids) >= 2 * threads:  # forked workers (numpy holds the GIL) write in place
        with ProcessPoolExecutor(max_workers=threads, mp_context=mp.get_context("fork")) as ex:
            res = list(ex.map(_shard_job, jobs, chunksize=1))
    else:
        res = [_shard_job(j) for j in jobs]
    load = np.zeros((m, J), dtype=np.float64)
    nnz = 0
    for (cfg_, cid, lo, hi, raw, so), (n, ld) in zip(jobs, res):  # compaction, left to right (nnz <= raw)
        if raw != nnz:
            _SH["dest"][nnz:nnz + n] = _SH["dest"][raw:raw + n]
            _SH["c"][nnz:nnz + n] = _SH["c"][raw:raw + n]
            _SH["a"][:, nnz:nnz + n] = _SH["a"][:, raw:raw + n]
        nnz += n
        load += ld
    lens = _SH.pop("lens")
    dest, c, a = _SH.pop("dest")[:nnz], _SH.pop("c")[:nnz], _SH.pop("a")
    a = a[:, :nnz] if m == 1 else np.ascontiguousarray(a[:, :nnz])
    row_ptr = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    inst = Instance(num_sources=int(lens.size), num_dests=J, num_families=m, row_ptr=row_ptr,
                    dest=dest, a=a, c=c, b=None, source_offset=src_begin)
    return inst, load


def _greedy_load(lens, dest, a, J):
    m = a.shape[0]
    load = np.zeros((m, J), dtype=np.float64)
    if dest.size == 0:
        return load
    src = np.repeat(np.arange(lens.size), lens)
    starts = np.zeros(lens.size, dtype=np.int64)
    np.cumsum(lens[:-1], out=starts[1:])
    nz = lens > 0
    for k in range(m):
        bmax = np.maximum.reduceat(a[k], starts[nz])
        full = np.zeros(lens.size, dtype=np.float32)
        full[nz] = bmax
        hit = np.flatnonzero(a[k] == full[src])
        _, first = np.unique(src[hit], return_index=True)
        sel = hit[first]
        load[k] += np.bincount(dest[sel], weights=a[k][sel].astype(np.float64), minlength=J)
    return load


def capacities(cfg: GenConfig, total_load: np.ndarray) -> np.ndarray:
    """b_kj = rho_kj (l_kj + eps), float32, family-major."""
    dp = dest_params(cfg)
    return (dp["rho"] * (total_load + cfg.slack_eps)).astype(np.float32).reshape(-1)


def generate(cfg: GenConfig, threads: int = 8) -> Instance:
    """The whole instance (single process)."""
    inst, load = generate_shard(cfg, 0, cfg.num_sources, threads=threads)
    inst.b = capacities(cfg, load)
    return inst
