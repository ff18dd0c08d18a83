// Fused dual-gradient pass (K1).  Included once per family count M and
// polytope kind by grad_m<M>_k<KIND>.cu (DL_GRAD_M, DL_GRAD_KIND); launch_fused_grad (grad.cu)
// dispatches on (m, kind).
//
// One persistent CTA per SM (16 warps).  For every source block i:
//   s_ij = c_ij + sum_k a_kij lambda_kj                 (reduced cost)
//   y_ij = -s_ij / gamma_i,  gamma_i = gamma v_i^2
//   x_i  = Pi_{C_i}(y_i) = clip(phi - d_ij, 0, u),  d_ij = (s_ij - min_j s_ij)/gamma_i,
//          phi the threshold of the block polytope (R1, R7)
//   acc[k*J + j] += a_kij x_ij   (fp64 red.global, only where x_ij > 0)
//   acc[mJ+0] += c_ij x_ij, acc[mJ+1] += gamma_i/2 x_ij^2, acc[mJ+2] += [x_ij > 0]
// into the CTA's own copy of the accumulator (launch_partial_sum adds the copies): reductions from
// every SM onto one shared m*J array put the B200 into a state where the whole pass streams ~1.6x
// slower; CTA-private rows do not.
//
// Work = the tile list of the layout (plan.cpp).
//  Phase 1 (blocks >= 256 entries, buckets >= 9): multi-warp groups (16/8/4/2 warps for
//   buckets >=12/11/10/9) read the block from global memory; d in an fp64 scratch.
//  Phase 2 (short blocks): every warp pulls tiles independently; a tile's dest / c / a_k
//   arrays arrive by cp.async.bulk (TMA bulk copy) into a per-warp double buffer with an
//   mbarrier.  A tile's blocks are worked by groups of G = 1..32 lanes (G = 2^(t-3) for
//   bucket t), <= 8 entries per lane.
//   Fast filter: s is first formed in fp32 (one FMA per family) and only entries with
//   s32 - min s32 <= gamma_i r + slack can have x > 0 on the simplex (active d < phi <= r),
//   resp. s32 < slack on the box (slack: the block's fp32 rounding bound).  Those candidates alone are re-formed exactly in fp64
//   (products of fp32 are exact in fp64) and the threshold is solved in fp64 (Michelot,
//   one or two candidates per lane: shuffle reductions over the group).  Box-cut blocks
//   and groups with more candidates take the generic exact path: fp64 d for every entry,
//   safeguarded Newton on the piecewise-linear F(phi) = sum clip(phi - d, 0, u) with an
//   Illinois-secant / bisection fallback.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "internal.h"

namespace dl {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCmax = 8;   // candidates per lane on the register fast path
constexpr int kRcpN = 64;  // 1/n table for the Michelot threshold (sum/n within 1 ulp)
__constant__ double c_rcp[kRcpN + 1] = {
    0.0,        1.0,        1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,  1.0 / 6,  1.0 / 7,  1.0 / 8,  1.0 / 9,  1.0 / 10,
    1.0 / 11,   1.0 / 12,   1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19, 1.0 / 20, 1.0 / 21,
    1.0 / 22,   1.0 / 23,   1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28, 1.0 / 29, 1.0 / 30, 1.0 / 31, 1.0 / 32,
    1.0 / 33,   1.0 / 34,   1.0 / 35, 1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39, 1.0 / 40, 1.0 / 41, 1.0 / 42, 1.0 / 43,
    1.0 / 44,   1.0 / 45,   1.0 / 46, 1.0 / 47, 1.0 / 48, 1.0 / 49, 1.0 / 50, 1.0 / 51, 1.0 / 52, 1.0 / 53, 1.0 / 54,
    1.0 / 55,   1.0 / 56,   1.0 / 57, 1.0 / 58, 1.0 / 59, 1.0 / 60, 1.0 / 61, 1.0 / 62, 1.0 / 63, 1.0 / 64};
#define kInfF __int_as_float(0x7f800000)
#define kInfD __longlong_as_double(0x7ff0000000000000LL)

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Streaming variant: the tile arrays are read once per pass, so they are loaded with an L2 evict-first
// policy and do not push the CTA accumulator copies, tile descriptors and duals out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                    uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void red_add_f64(double* a, double v) {  // fire-and-forget fp64 reduction
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- group reductions
// Butterflies over aligned groups of G lanes (G a power of two <= 32): every lane of
// a group ends with bitwise the same value (a+b == b+a in IEEE arithmetic).
template <class T>
__device__ __forceinline__ T gsum(T v, int G) {
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
template <class T>
__device__ __forceinline__ T gmin(T v, int G) {
  for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
template <class T>
__device__ __forceinline__ T gmax(T v, int G) {
  for (int o = 1; o < G; o <<= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// ---------------------------------------------------------------- exact threshold solver
// F(phi) = u nC + phi nM - sM with M = {phi-u < d < phi}, C = {d <= phi-u} (fp64).
struct Sums {
  double nM, sM, nC;
};
__device__ __forceinline__ double capsum(double u, double nC) { return nC > 0.0 ? u * nC : 0.0; }
__device__ __forceinline__ double Fval(double phi, double u, const Sums& s) {
  return capsum(u, s.nC) + phi * s.nM - s.sM;
}

struct Solver {
  double lo, hi, Flo, Fhi, phi;
  int side;   // last bracket end replaced: +1 hi, -1 lo (Illinois)
  bool done;
  bool free;  // theta = 0: the clamp alone is feasible, phi = phi_free
};

// Start at hi0 (F(hi0) >= r unless hi0 == phi_free); bracket [0, hi0] (F(0) = 0 <= r as d >= 0).
__device__ __forceinline__ void solver_start(Solver& S, double r, double u, double phi_free, const Sums& s0,
                                             double hi0) {
  const double F = Fval(hi0, u, s0);
  S.lo = 0.0;
  S.Flo = 0.0;
  S.hi = hi0;
  S.Fhi = F;
  S.phi = hi0;
  S.side = 0;
  S.done = false;
  S.free = false;
  if (hi0 == phi_free && F <= r) {
    S.phi = phi_free;
    S.done = true;
    S.free = true;
  } else if (F == r) {
    S.done = true;
  }
}
// Newton step from the partition at S.phi; falls back to Illinois secant / bisection.
__device__ __forceinline__ double solver_candidate(Solver& S, double r, double u, const Sums& s) {
  double cand = s.nM > 0.0 ? (r - capsum(u, s.nC) + s.sM) / s.nM : __longlong_as_double(0x7ff8000000000000LL);
  if (!(cand > S.lo && cand < S.hi)) {
    cand = S.Fhi > S.Flo ? S.lo + (r - S.Flo) * (S.hi - S.lo) / (S.Fhi - S.Flo) : 0.5 * (S.lo + S.hi);
    if (!(cand > S.lo && cand < S.hi)) cand = 0.5 * (S.lo + S.hi);
  }
  if (cand == S.phi) S.done = true;
  return cand;
}
__device__ __forceinline__ void solver_update(Solver& S, double r, double u, const Sums& s) {
  const double F = Fval(S.phi, u, s);
  if (F > r) {
    S.hi = S.phi;
    S.Fhi = F;
    if (S.side == 1) S.Flo = r + 0.5 * (S.Flo - r);  // Illinois: lo retained twice
    S.side = 1;
  } else if (F < r) {
    S.lo = S.phi;
    S.Flo = F;
    if (S.side == -1) S.Fhi = r + 0.5 * (S.Fhi - r);
    S.side = -1;
  } else {
    S.done = true;
  }
  if (!(S.hi - S.lo > 4e-16 * fabs(S.hi))) S.done = true;
}

// ---------------------------------------------------------------- shared memory
struct SmemHead {
  uint64_t mbar[kWarps][2];       // data stages (tile arrays + block offsets)
  uint64_t mbar_desc[kWarps][2];  // descriptor-chunk slots
  double red[2][kWarps][3];
  double rcp[kRcpN + 1];          // 1/n, n = 0..kRcpN (copied from c_rcp: divergent n, no constant-bank replays)
  int32_t slot[16];
  int32_t ccount[16];             // candidate-list fill of each big-block group (phase 1)
};
static_assert(sizeof(SmemHead) <= 2048, "head fits the fixed smem reserve");

// The accumulator copy of this CTA: copies are assigned to runs of consecutive SM ids (one per SM when
// there are as many copies as CTAs), so that a copy shared by several CTAs is shared by neighbouring SMs.
__device__ __forceinline__ int copy_of(const GradArgs& p) {
  if (p.acc_copies >= (int)gridDim.x) return blockIdx.x;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  return (int)min((uint32_t)p.acc_copies - 1u, sm * (uint32_t)p.acc_copies / max(1u, (uint32_t)p.num_sms));
}

template <int M, int LM, bool WX>
struct Ctx {
  const GradArgs& p;
  const float* lam_s;  // duals staged in shared memory (LM != kLamGlobal)
  uint32_t lam_sa;     // their shared-window address
  const float* lam_g;  // all duals in global memory
  int J, H;            // destinations; labels staged per family (kLamHot)
  double* acc;         // this CTA's accumulator copy
  double gamma, invgamma;
  double cx = 0.0, reg = 0.0;
  float nx = 0.f;
  __device__ Ctx(const GradArgs& pp, const float* ls, double g)
      : p(pp), lam_s(ls), lam_sa(ls ? smem_u32(ls) : 0u), lam_g(pp.lam), J(pp.J), H(pp.lam_hot), acc(pp.acc + (size_t)copy_of(pp) * pp.acc_stride),
        gamma(g),
        invgamma(1.0 / g) {}

  // dual of family f at destination label j: shared memory (all, or the hot labels [0, H) of
  // the popularity order, R15) or global memory (L2-resident m*J floats)
  // (hot: shared-memory load for labels < H, read-only global load otherwise -- two predicated loads,
  // never a generic-address load, whose shared-window test costs ~10 instructions per lookup)
  // The staged duals are read with 32-bit shared-window addresses from a base kept in a register (a
  // generic pointer into shared memory made the compiler re-derive the window base -- S2R
  // SR_CgaCtaId, MOV, LEA -- before many lookups).  The asm is not volatile: the duals are written
  // once before the CTA barrier and never again, so the loads may be scheduled freely.
  __device__ __forceinline__ float lds(uint32_t a) const {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
  }
  __device__ __forceinline__ float lam(int f, int j) const {
    if constexpr (LM == kLamSmem) return lds(lam_sa + 4u * (uint32_t)(f * J + j));
    if constexpr (LM == kLamHot) {
      float v;
      if (j < H) v = lds(lam_sa + 4u * (uint32_t)(f * H + j));
      else v = __ldg(lam_g + f * J + j);
      return v;
    }
    return __ldg(lam_g + f * J + j);
  }
  // contribution of one positive x (fp64) to A x, the objective scalars and x_out
  __device__ __forceinline__ void emit(int j, float cval, const float* av, double x, double vs, int b, int e) {
#pragma unroll
    for (int f = 0; f < M; ++f) red_add_f64(acc + (size_t)f * p.J + j, (double)av[f] * x);
    cx += (double)cval * x;
    reg += 0.5 * gamma * vs * x * x;
    nx += 1.f;
    if constexpr (WX) p.x_out[__ldg(p.orig_off + b) + e] = (float)x;
  }
};

// ---------------------------------------------------------------- phase 1: big blocks
struct BigGroup {
  int gw, G, gtid, warp0, bar, lane, warp;
  int rb = 0;
  SmemHead* head;
  __device__ __forceinline__ void sync() { named_bar(bar, G); }
  // reduce up to 3 doubles with op (0 sum, 1 min, 2 max); deterministic order
  template <int N>
  __device__ __forceinline__ void reduce(double (&v)[N], int op) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      for (int o = 16; o > 0; o >>= 1) {
        double w = __shfl_xor_sync(kFull, v[i], o);
        v[i] = op == 0 ? v[i] + w : (op == 1 ? fmin(v[i], w) : fmax(v[i], w));
      }
    }
    const int b = rb;
    rb ^= 1;
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < N; ++i) head->red[b][warp][i] = v[i];
    sync();
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double t = head->red[b][warp0][i];
      for (int w = 1; w < gw; ++w) {
        const double q = head->red[b][warp0 + w][i];
        t = op == 0 ? t + q : (op == 1 ? fmin(t, q) : fmax(t, q));
      }
      v[i] = t;
    }
  }
};

template <int M, int LM, bool WX>
__device__ __forceinline__ double score_global(const Ctx<M, LM, WX>& C, int64_t e) {
  const GradArgs& p = C.p;
  const int j = __ldg(p.dest + e);
  double s = (double)__ldg(p.c + e);
#pragma unroll
  for (int f = 0; f < M; ++f) s = fma((double)__ldg(p.a + f * p.a_stride + e), (double)C.lam(f, j), s);
  return s;
}

template <int M, int LM, bool WX>
__device__ void big_block(Ctx<M, LM, WX>& C, BigGroup& g, const Tile& tl, double* scr) {
  const GradArgs& p = C.p;
  const int len = tl.nnz;
  const int64_t off = tl.off;
  const int b = tl.b0;
  const double r = p.r, u = p.u;
  // pass 1: exact minimum reduced cost
  double mn[1] = {DBL_MAX};
#pragma unroll 4
  for (int e = g.gtid; e < len; e += g.G) mn[0] = fmin(mn[0], score_global(C, off + e));
  g.reduce(mn, 1);
  const double smin = mn[0];
  const double vs = p.vsq ? (double)__ldg(p.vsq + b) : 1.0;
  const double ginv = p.vsq ? C.invgamma * (double)__ldg(p.vinv + b) : C.invgamma;
  const double phi_free = -smin * ginv;
  // pass 2: d = (s - smin)/gamma_i into the scratch (own entries only)
  double mx[1] = {-DBL_MAX};
#pragma unroll 4
  for (int e = g.gtid; e < len; e += g.G) {
    const double d = (score_global(C, off + e) - smin) * ginv;
    scr[e] = d;
    mx[0] = fmax(mx[0], d);
  }
  double phi = phi_free;
  bool free = true;
  if (p.kind != DL_PROJ_BOX) {
    if (p.kind == DL_PROJ_BOXCUT) g.reduce(mx, 2);
    auto eval = [&](double ph) {
      double v[3] = {0.0, 0.0, 0.0};
      for (int e = g.gtid; e < len; e += g.G) {
        const double d = scr[e];
        if (d < ph) {
          if (d > ph - u) {
            v[0] += 1.0;
            v[1] += d;
          } else {
            v[2] += 1.0;
          }
        }
      }
      g.reduce(v, 0);
      return Sums{v[0], v[1], v[2]};
    };
    const double hi0 = p.kind == DL_PROJ_SIMPLEX ? fmin(phi_free, r) : fmin(phi_free, mx[0] + u);
    Solver S;
    Sums cur = eval(hi0);
    solver_start(S, r, u, phi_free, cur, hi0);
    for (int it = 0; it < 200 && !S.done; ++it) {
      const double cand = solver_candidate(S, r, u, cur);
      if (S.done) break;
      S.phi = cand;
      cur = eval(S.phi);
      solver_update(S, r, u, cur);
    }
    phi = S.phi;
    free = S.free;
  }
  for (int e = g.gtid; e < len; e += g.G) {
    const double d = scr[e];
    const double x = free ? fmin(fmax(phi_free - d, 0.0), u) : fmin(fmax(phi - d, 0.0), u);
    if (x > 0.0) {
      const int j = __ldg(p.dest + off + e);
      float av[M];
#pragma unroll
      for (int f = 0; f < M; ++f) av[f] = __ldg(p.a + f * p.a_stride + off + e);
      C.emit(j, __ldg(p.c + off + e), av, x, vs, b, e);
    }
  }
  g.sync();  // scratch reuse by the next block of this group
}

// ---------------------------------------------------------------- phase 2: small tiles
template <int M, int LM, bool WX>
__device__ __forceinline__ double score_smem(const Ctx<M, LM, WX>& C, const int32_t* sd, const float* sc,
                                             const float* sa, int cap, int ee) {
  const int j = sd[ee];
  double s = (double)sc[ee];
#pragma unroll
  for (int f = 0; f < M; ++f) s = fma((double)sa[f * cap + ee], (double)C.lam(f, j), s);
  return s;
}

template <int M, int LM, bool WX>
__device__ __forceinline__ void emit_smem(Ctx<M, LM, WX>& C, const int32_t* sd, const float* sc, const float* sa,
                                          int cap, int ee, double x, double vs, int b, int e) {
  float av[M];
#pragma unroll
  for (int f = 0; f < M; ++f) av[f] = sa[f * cap + ee];
  C.emit(sd[ee], sc[ee], av, x, vs, b, e);
}

// Compile-time group reductions (G lanes, aligned groups inside the warp).
template <int G, class T>
__device__ __forceinline__ T tsum(T v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
template <int G, class T>
__device__ __forceinline__ T tmin(T v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
template <int G, class T>
__device__ __forceinline__ T tmax(T v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
// number of set predicates over the group's lanes (one vote)
template <int G>
__device__ __forceinline__ int tcount(bool pred, uint32_t gmask) {
  return __popc(__ballot_sync(kFull, pred) & gmask);
}

// Michelot in fp64 by one warp on up to 8 candidates per lane (d64[c] valid where bit c of vm is set):
// phi* of F(phi) = sum max(phi - d, 0) = r over the candidates, threshold min(phi_free, phi*) (theta = 0
// exactly when phi_free <= phi*); a single candidate gets x = min(phi_free, r).  emit(c, x) for x > 0.
template <class EmitF>
__device__ __forceinline__ void warp_michelot(const double (&d64)[8], uint32_t vm, double r, double phi_free,
                                              const double* rcp, EmitF&& emit) {
  // |S| by one integer warp reduction per iteration (lane counts), 1/|S| from the shared table
  // (within 1 ulp) up to kRcpN; the fp64 sum only when |S| changed
  const int nT = (int)__reduce_add_sync(kFull, (unsigned)__popc(vm));
  const int pmax = 32 - (int)__reduce_min_sync(kFull, (unsigned)__clz(vm));  // highest slot in use + 1
  auto inv = [&](int n) { return n <= kRcpN ? rcp[n] : 1.0 / (double)n; };
  double sl = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (vm >> c & 1u) sl += d64[c];
  double phi = (r + tsum<32>(sl)) * inv(max(nT, 1));
  int cprev = nT;
  for (int it = 0; it < 300 && nT > 1; ++it) {
    int cl = 0;
    double s2 = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < pmax) {
        const bool in = (vm >> c & 1u) && d64[c] < phi;
        cl += in;
        if (in) s2 += d64[c];
      }
    const int cnt = (int)__reduce_add_sync(kFull, (unsigned)cl);
    if (cnt == cprev || cnt == 0) break;
    cprev = cnt;
    phi = (r + tsum<32>(s2)) * inv(cnt);
  }
  const double ph = nT == 1 ? phi_free : fmin(phi_free, phi);
  const double cap_x = nT == 1 ? r : kInfD;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (vm >> c & 1u) {
      const double x = fmin(fmax(ph - d64[c], 0.0), cap_x);
      if (x > 0.0) emit(c, x);
    }
}

// Big simplex block (>= 256 entries) by a multi-warp group, candidate version of big_block: pass 1
// streams the block from global memory (coalesced) for the fp32 minimum; pass 2 re-streams it (L2)
// and pushes the entries inside the candidate window (as small_tile) to a shared list; the group's
// first warp then runs warp_michelot on the list (<= 256 candidates; more -> big_block, exact generic).
template <int M, int LM, bool WX>
__device__ void big_block_simplex(Ctx<M, LM, WX>& C, BigGroup& g, const Tile& tl, double* scr, int scr_cap,
                                  double* scr_generic) {
  const GradArgs& p = C.p;
  const int len = tl.nnz;
  const int64_t off = tl.off;
  const int b = tl.b0;
  const unsigned Jm1 = (unsigned)p.J - 1u;
  int32_t* list = reinterpret_cast<int32_t*>(scr);
  const int list_cap = min(256, 2 * scr_cap);
  int32_t* cnt_s = &g.head->ccount[g.bar];
  // U entries per thread per step, loads issued before use (the lambda gathers may miss to L2)
  constexpr int U = 8;
  auto scores = [&](int e0, float (&sv)[U], float (&mg)[U]) {
    int j[U];
    float cv[U], av[M][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = min(e0 + u * g.G, len - 1);
      j[u] = (int)min((unsigned)__ldg(p.dest + off + e), Jm1);
      cv[u] = __ldg(p.c + off + e);
#pragma unroll
      for (int f = 0; f < M; ++f) av[f][u] = __ldg(p.a + f * p.a_stride + off + e);
    }
    float lv[M][U];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int f = 0; f < M; ++f) lv[f][u] = C.lam(f, j[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      sv[u] = cv[u];
      mg[u] = fabsf(cv[u]);
#pragma unroll
      for (int f = 0; f < M; ++f) {
        sv[u] = fmaf(av[f][u], lv[f][u], sv[u]);
        if constexpr (M > 1) mg[u] = fmaf(fabsf(av[f][u]), fabsf(lv[f][u]), mg[u]);
      }
      if (e0 + u * g.G >= len) sv[u] = kInfF, mg[u] = 0.f;
    }
  };
  float lmin = kInfF, lmag = 0.f;
  for (int e0 = g.gtid; e0 < len; e0 += U * g.G) {
    float sv[U], mg[U];
    scores(e0, sv, mg);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      lmin = fminf(lmin, sv[u]);
      lmag = fmaxf(lmag, mg[u]);
    }
  }
  if (g.gtid == 0) *cnt_s = 0;  // ordered before pass 2 by the barrier of the reduce
  double v[2] = {(double)lmin, -(double)lmag};
  g.reduce(v, 1);
  const float ref = (float)v[0];
  const double vs = p.vsq ? (double)__ldg(p.vsq + b) : 1.0;
  const double ginv = p.vsq ? C.invgamma * (double)__ldg(p.vinv + b) : C.invgamma;
  const float gr = (float)(p.r * C.gamma * vs);
  const float slack = M == 1 ? 4.7683716e-7f * (fabsf(ref) + gr) : 2.3841858e-7f * (M + 1) * (float)(-v[1]);
  const float T = ref + (gr * 1.000001f + slack);
  const unsigned lt_mask = (1u << g.lane) - 1u;
  for (int b0 = 0; b0 < len; b0 += U * g.G) {  // warp-uniform trip count
    float sv[U], mg[U];
    scores(b0 + g.gtid, sv, mg);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = b0 + g.gtid + u * g.G;
      const bool cand = sv[u] <= T;  // +inf past the block
      const unsigned m = __ballot_sync(kFull, cand);
      if (m) {
        int base = 0;
        if (g.lane == 0) base = atomicAdd(cnt_s, __popc(m));
        base = __shfl_sync(kFull, base, 0);
        if (cand) {
          const int pos = base + __popc(m & lt_mask);
          if (pos < list_cap) list[pos] = e;
        }
      }
    }
  }
  g.sync();
  const int nc = *cnt_s;
  if (nc > list_cap) {  // candidate overflow: exact generic path
    g.sync();
    big_block<M, LM, WX>(C, g, tl, scr_generic);
    return;
  }
  if (g.warp == g.warp0) {
    const double refd = (double)ref;
    double d64[8];
    int ee[8];
    uint32_t vm = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      d64[c] = kInfD;
      ee[c] = 0;
      const int i = g.lane + 32 * c;
      if (i < nc) {
        ee[c] = list[i];
        d64[c] = (score_global(C, off + ee[c]) - refd) * ginv;
        vm |= 1u << c;
      }
    }
    warp_michelot(d64, vm, p.r, -refd * ginv, g.head->rcp, [&](int c, double x) {
      const int64_t e = off + ee[c];
      float av[M];
#pragma unroll
      for (int f = 0; f < M; ++f) av[f] = __ldg(p.a + f * p.a_stride + e);
      C.emit(__ldg(p.dest + e), __ldg(p.c + e), av, x, vs, b, ee[c]);
    });
  }
  g.sync();  // the list and its counter are reused by the group's next block
}

// fp32 threshold solver state for the generic small path (partition only; the final
// threshold is recomputed in fp64 from the partition).
struct SolverF {
  float lo, hi, Flo, Fhi, phi;
  int side;
  bool done, free;
};
struct SumsF {
  float nM, sM, nC;
};
__device__ __forceinline__ float capsumf(float u, float nC) { return nC > 0.f ? u * nC : 0.f; }

// ---- generic exact solve for one round (box-cut, or a group with > 4 G simplex candidates).
// Candidates cm (bit k: entry q + k G of the block), frame origin ref (fl32 min of s for the
// simplex, the K-th smallest s for box-cut).  d = fl32((s - ref)/gamma_i) with s exact, so every
// entry near a breakpoint is O(max(r, u)) in this frame; a safeguarded Newton in fp32 (Illinois
// secant / bisection fallback) finds the partition, then Newton steps in fp64 on the exact
// partition (exact d recomputed from shared memory) give phi = (r - u|C| + sum_M d)/|M|.
// Slot k of lane q (group of G lanes) -> block-relative entry: strided (q + k G), or, in the
// float4 layout of the small-tile path, component k&3 of the lane's (k>>2)-th float4 q + (k>>2) G.
template <int LG, bool V4>
__device__ __forceinline__ int slot_entry(int q, int k) {
  return V4 ? 4 * (q + (k >> 2) * (1 << LG)) + (k & 3) : q + k * (1 << LG);
}

template <int M, int LM, bool WX, int LG, int E, bool V4>
__device__ __forceinline__ void generic_round(Ctx<M, LM, WX>& C, const int32_t* sd, const float* sc,
                                              const float* sa, int cap, int q, int start, bool active, int b,
                                              double vs, double ginv, uint32_t cm, float ref, float (&d)[E]) {
  constexpr int G = 1 << LG;
  const GradArgs& p = C.p;
  const int kind = p.kind;
  const double r = p.r, u = p.u;
  const float rf = p.r, uf = p.u;
  const double refd = (double)ref;
  auto dexact = [&](int k) { return (score_smem(C, sd, sc, sa, cap, start + slot_entry<LG, V4>(q, k)) - refd) * ginv; };
  // d in fp32 from the caller's fp32 scores (in place): only the partition search uses it; the
  // fp64 Newton steps below re-derive exact d from shared memory and settle any boundary entry
  const float ginvf = (float)ginv;
  float dmax = -kInfF, dmn = kInfF;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    d[k] = (cm >> k & 1u) ? (d[k] - ref) * ginvf : kInfF;
    if (cm >> k & 1u) {
      dmax = fmaxf(dmax, d[k]);
      dmn = fminf(dmn, d[k]);
    }
  }
  dmn = tmin<G>(dmn);
  const double phi_free64 = -refd * ginv;
  const float phi_free = (float)fmax(fmin(phi_free64, 1e30), -1e30);
  auto local = [&](float ph) {
    SumsF s{0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < E; ++k) {
      if (d[k] < ph) {
        if (d[k] > ph - uf) {
          s.nM += 1.f;
          s.sM += d[k];
        } else {
          s.nC += 1.f;
        }
      }
    }
    s.nM = tsum<G>(s.nM);
    s.sM = tsum<G>(s.sM);
    s.nC = tsum<G>(s.nC);
    return s;
  };
  const float hi0 = kind == DL_PROJ_SIMPLEX ? fminf(phi_free, dmn + rf) : fminf(phi_free, tmax<G>(dmax) + uf);
  SolverF S;
  S.done = true;
  S.free = true;
  S.phi = phi_free;
  S.lo = S.hi = S.Flo = S.Fhi = 0.f;
  S.side = 0;
  SumsF cur = local(hi0);
  if (active) {
    const float F = capsumf(uf, cur.nC) + hi0 * cur.nM - cur.sM;
    S.lo = dmn;  // F(d_min) = 0
    S.Flo = 0.f;
    S.hi = hi0;
    S.Fhi = F;
    S.phi = hi0;
    S.free = hi0 == phi_free && F <= rf;
    S.done = S.free || F == rf;
  }
  for (int it = 0; it < 200 && __any_sync(kFull, !S.done); ++it) {
    if (!S.done) {
      float cand = cur.nM > 0.f ? (rf - capsumf(uf, cur.nC) + cur.sM) / cur.nM : __int_as_float(0x7fc00000);
      if (!(cand > S.lo && cand < S.hi)) {
        cand = S.Fhi > S.Flo ? S.lo + (rf - S.Flo) * (S.hi - S.lo) / (S.Fhi - S.Flo) : 0.5f * (S.lo + S.hi);
        if (!(cand > S.lo && cand < S.hi)) cand = 0.5f * (S.lo + S.hi);
      }
      if (cand == S.phi) S.done = true;
      else S.phi = cand;
    }
    const bool want = !S.done;
    if (!__any_sync(kFull, want)) break;
    cur = local(S.phi);
    if (want) {
      const float F = capsumf(uf, cur.nC) + S.phi * cur.nM - cur.sM;
      if (F > rf) {
        S.hi = S.phi;
        S.Fhi = F;
        if (S.side == 1) S.Flo = rf + 0.5f * (S.Flo - rf);
        S.side = 1;
      } else if (F < rf) {
        S.lo = S.phi;
        S.Flo = F;
        if (S.side == -1) S.Fhi = rf + 0.5f * (S.Fhi - rf);
        S.side = -1;
      } else {
        S.done = true;
      }
      if (!(S.hi - S.lo > 2.4e-7f * fabsf(S.hi))) S.done = true;
    }
  }
  // theta = 0 decided exactly: F(phi_free) = sum clip(phi_free - d, 0, u) <= r in fp64
  double ff = 0.0;
#pragma unroll
  for (int k = 0; k < E; ++k)
    if (cm >> k & 1u) ff += fmin(fmax(phi_free64 - dexact(k), 0.0), u);
  ff = tsum<G>(ff);
  const bool free64 = phi_free64 <= 1e30 && ff <= r;
  if (S.free && !free64) S.phi = phi_free;  // the fp32 test was too optimistic: Newton from phi_free
  // fp64 phase on the exact d: safeguarded Newton on the piecewise-linear F, started at the fp32
  // result, with a bracket lo < phi* <= hi kept from fp64 evaluations (F(lo) < r < F(hi)); ends when
  // F(phi) == r (a flat piece included) or the bracket/step is at fp64 resolution.  Membership is
  // never decided in fp32 here (an fp32 partition can put phi a few ulps(d32) inside a neighbouring
  // piece, PAPER.md:125-134 readings R1/R7).
  // initial bracket: F(lo) = 0 below every d; F(hi) >= r (simplex: the minimum entry alone reaches
  // r at d_min + r; box-cut: >= K = ceil(r/u) entries capped at d_(K) + u <= d_max + u)
  const double marg = 1.0 + 1e-6 * (fabs((double)dmn) + fabs(refd) * ginv + fabs((double)hi0));
  double lo = (double)dmn - marg;
  double hi = (double)fmaxf(hi0, S.phi) + marg;
  double ph = free64 ? phi_free64 : (double)S.phi;
  bool fin = !active || free64;
  for (int it = 0; it < 40 && __any_sync(kFull, !fin); ++it) {
    double sM = 0.0;
    float nM = 0.f, nC = 0.f;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      if (cm >> k & 1u) {
        const double dd = dexact(k);
        if (dd < ph) {
          if (dd > ph - u) {
            nM += 1.f;
            sM += dd;
          } else {
            nC += 1.f;
          }
        }
      }
    }
    nM = tsum<G>(nM);
    nC = tsum<G>(nC);
    sM = tsum<G>(sM);
    if (!fin) {
      const double F = (nC > 0.f ? u * nC : 0.0) + (nM > 0.f ? ph * nM - sM : 0.0);
      if (F == r) {
        fin = true;
      } else {
        if (F > r) hi = ph;
        else lo = ph;
        double np = nM > 0.f ? (r - (nC > 0.f ? u * nC : 0.0) + sM) / nM : __longlong_as_double(0x7ff8000000000000LL);
        if (!(np > lo && np < hi)) np = 0.5 * (lo + hi);
        if (np == ph || !(hi - lo > 4e-16 * fmax(fabs(hi), fabs(lo)))) fin = true;
        ph = np;
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if (cm >> k & 1u) {
      const double x = fmin(fmax(ph - dexact(k), 0.0), u);
      if (x > 0.0) {
        const int e = slot_entry<LG, V4>(q, k);
        emit_smem(C, sd, sc, sa, cap, start + e, x, vs, b, e);
      }
    }
  }
}

// Short blocks of one tile (buckets < kBigBucket) for the BOX and BOX-CUT polytopes, G = 2^LG
// lanes per block, NG = 32/G blocks per round, E entries (slots) per lane (E G > every length of
// the bucket).  Groups with more candidates than the register path holds take the generic exact
// solve (generic_round).  (Simplex tiles: small_tile_simplex below.)
template <int M, int LM, bool WX, int LG, int E, bool GEN>
__device__ void small_tile(Ctx<M, LM, WX>& C, const Tile& tl, const char* stage, int lane,
                           const uint16_t* rel_s, uint16_t* cand_s, const double* rcp_s) {
  constexpr int G = 1 << LG;
  constexpr int NG = 32 >> LG;
  // candidates per lane on the register path.  OWN (E <= 8 slots per lane, blocks < 32 entries): a
  // lane's candidates are its own slots, no shared list; otherwise the group's candidates are
  // compacted into a shared list, <= 4 per lane (more: generic_round)
  constexpr bool OWN = E <= 8;
  constexpr int CAP = OWN ? E : 4;
  const GradArgs& p = C.p;
  const int cap = p.tile_cap;
  const int32_t* sd = reinterpret_cast<const int32_t*>(stage);
  const float* sc = reinterpret_cast<const float*>(stage) + cap;
  const float* sa = sc + cap;  // family f at sa + f*cap
  const int gi = lane >> LG, q = lane & (G - 1);
  const uint32_t gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << (gi * G);
  const int nrounds = (tl.nb + NG - 1) / NG;
  const int kind = p.kind;
  for (int rd = 0; rd < nrounds; ++rd) {
    const int bb = rd * NG + gi;
    const bool active = bb < tl.nb;
    const int b = tl.b0 + bb;
    // block bounds: streamed into shared memory with the tile ({rel_0..rel_{nb-1},
    // nnz}), or read from global memory for tiles with many blocks
    int start = 0, end = 0;
    if (active) {
      if (tl.rel_off >= 0) {
        start = rel_s[bb];
        end = rel_s[bb + 1];
      } else {
        start = (int)__ldg(p.blk_rel + b);
        end = bb + 1 < tl.nb ? (int)__ldg(p.blk_rel + b + 1) : tl.nnz;
      }
    }
    double vs = 1.0, ginv = C.invgamma;  // gamma_i = gamma v_i^2
    if (p.vsq) {
      if (active) {
        vs = (double)__ldg(p.vsq + b);
        ginv = C.invgamma * (double)__ldg(p.vinv + b);
      }
    }
    // ---- fp32 pass: s32 = fl(c + sum_f a_f lambda_f) (one FMA per family) for every slot; slot k
    // of lane q is entry q + k G of the block (consecutive lanes read consecutive words: no bank
    // conflicts on the stage); slots past the block end are +inf.
    float s32[E];
    float lmin = kInfF, lmag = 0.f;
    {
      const int lim = (end - start) - q;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int ee = start + q + k * G;
        const bool in = k * G < lim;
        const int j = in ? sd[ee] : 0;  // reads past the tile stay inside shared memory (tail pad)
        float sv = in ? sc[ee] : kInfF, mg = fabsf(sv);
#pragma unroll
        for (int f = 0; f < M; ++f) {
          const float a_ = in ? sa[f * cap + ee] : 0.f, lv = C.lam(f, j);
          sv = fmaf(a_, lv, sv);
          if constexpr (M > 1) mg = fmaf(fabsf(a_), fabsf(lv), mg);
        }
        s32[k] = sv;
        lmin = fminf(lmin, sv);
        if constexpr (M > 1) lmag = sv < kInfF ? fmaxf(lmag, mg) : lmag;
      }
    }
    // ---- candidates: entries that can have x > 0.  M = 1: one rounding, |fl(s) - s| <= 2^-24 |s|;
    // M > 1: |fl32(s) - s| <= M 2^-24 (|c| + sum_f |a_f lambda_f|) = M 2^-24 mag per entry.
    uint32_t cm = 0;
    if (kind == DL_PROJ_BOX) {  // x > 0  iff  s < 0: no coupling inside the block, x = clip(-s/gamma_i, 0, u)
      // M = 1: the rounding keeps the sign (s < 0 => fl(s) <= 0); M > 1: lane bound 2^-22 (M+1) mag
      const float slack = M == 1 ? 0.f : 2.3841858e-7f * (M + 1) * lmag;
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (s32[k] <= slack) cm |= 1u << k;
      if (!active) cm = 0;
      while (cm) {
        const int k = __ffs(cm) - 1;
        cm &= cm - 1;
        const int e = slot_entry<LG, false>(q, k), ee = start + e;
        const double x = fmin(fmax(-score_smem(C, sd, sc, sa, cap, ee) * ginv, 0.0), (double)p.u);
        if (x > 0.0) emit_smem(C, sd, sc, sa, cap, ee, x, vs, b, e);
      }
      continue;
    }
    const double r = p.r;
    // candidate window: entries that can be active.  Simplex: active d < phi <= r, i.e.
    // s - s_min < gamma_i r; frame origin ref = s_min.  Box-cut: active d < phi <= d_(K) + u,
    // K = ceil(r/u) (the K smallest at the cap already reach r); frame origin ref = s_(K).
    // The slack covers the two roundings of s_j - ref and of the threshold sum: M = 1: 2^-21
    // (|ref| + width) (>= 2.6x the bound 2^-24 (3 |ref| + 2 width)); M > 1: 2^-22 (M+1) max mag.
    const bool boxcut = GEN && kind == DL_PROJ_BOXCUT;
    const float slack_m = M == 1 ? 0.f : 2.3841858e-7f * (M + 1) * tmax<G>(lmag);
    float ref;
    if (boxcut) {
      const double u = p.u;
      const int K = (int)ceil(r / u);
      float sk = 0.f, cnt = 0.f;  // sk: K-th smallest s32 (or the largest, if fewer than K)
      uint32_t excl = 0;
      bool sat = !active;
      if (K <= 8) {
        for (int rnd = 0; rnd < 8 && __any_sync(kFull, !sat); ++rnd) {
          float ml = kInfF;
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (!(excl >> k & 1u)) ml = fminf(ml, s32[k]);
          const float m = tmin<G>(ml);
          float c = 0.f;
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (!(excl >> k & 1u) && s32[k] == m) {
              c += 1.f;
              excl |= 1u << k;
            }
          c = tsum<G>(c);
          if (!sat) {
            if (m == kInfF) {  // fewer than K entries: the sum cap cannot bind, all are candidates
              sat = true;
            } else {
              cnt += c;
              sk = m;
              if (cnt >= (float)K) sat = true;
            }
          }
        }
      }
      if (sat) {
        const float gu = (float)(u * C.gamma * vs);
        const float slack = M == 1 ? 4.7683716e-7f * (fabsf(sk) + gu) : slack_m;
        const float T = sk + (gu * 1.000001f + slack);
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (s32[k] <= T) cm |= 1u << k;
      } else {  // K > 8: every entry is a candidate
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (s32[k] < kInfF) cm |= 1u << k;
      }
      ref = sat ? sk : tmin<G>(lmin);
    } else {
      ref = tmin<G>(lmin);
      const float gr = (float)(r * C.gamma * vs);
      const float slack = M == 1 ? 4.7683716e-7f * (fabsf(ref) + gr) : slack_m;
      const float T = ref + (gr * 1.000001f + slack);
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (s32[k] <= T) cm |= 1u << k;
    }
    if (!active) cm = 0;
    // ---- compaction: the group's candidates (tile entry indices) are packed into a per-warp
    // shared list so that lane q of the group owns candidates q, q+G, .. (<= CAP G).
    const int nc = __popc(cm);
    int incl = nc;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o, G);
      if (q >= o) incl += v;
    }
    int T = __shfl_sync(kFull, incl, G - 1, G);  // candidates of the group
    if (!__all_sync(kFull, T <= CAP * G)) {  // many candidates: exact generic solve of the round
      generic_round<M, LM, WX, LG, E, false>(C, sd, sc, sa, cap, q, start, active, b, vs, ginv, cm, ref, s32);
      continue;
    }
    if constexpr (!OWN) {
      uint32_t m = cm;
      int o = gi * CAP * G + incl - nc;
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        cand_s[o++] = (uint16_t)(start + slot_entry<LG, false>(q, k));
      }
      __syncwarp();
    }
    // candidate slots to visit (warp-uniform): own slots -> the largest per-lane count
    const int pmax = OWN ? (int)__reduce_max_sync(kFull, (unsigned)nc)
                         : (int)((__reduce_max_sync(kFull, (unsigned)T) + G - 1) >> LG);
    const double refd = (double)ref;
    const double phi_free = -refd * ginv;  // x_free = max(phi_free - d, 0) = max(-s/gamma_i, 0)
    double d64[CAP];
    int ei[CAP];
    uint32_t mo = cm;  // OWN: the lane's remaining candidate slots, consumed in slot order
#pragma unroll
    for (int c = 0; c < CAP; ++c) {
      d64[c] = kInfD;
      ei[c] = -1;
      if (c < pmax) {
        const int idx = OWN ? c : q + c * G;
        if (idx < (OWN ? nc : T)) {
          int ee;
          if constexpr (OWN) {  // c-th candidate slot of the lane itself
            ee = start + slot_entry<LG, false>(q, __ffs(mo) - 1);
            mo &= mo - 1;
          } else {
            ee = cand_s[gi * CAP * G + idx];
          }
          d64[c] = (score_smem(C, sd, sc, sa, cap, ee) - refd) * ginv;
          ei[c] = ee;
        }
      }
    }
    if (boxcut) {
      // box-cut, exact on the candidates in fp64: theta = 0 when F(phi_free) <= r (F(phi) = sum
      // clip(phi - d, 0, u)); else the root of F(phi) = r by Newton on the current piece,
      // phi = (r - u |C| + sum_M d)/|M| (M = {phi - u < d < phi}, C = {d <= phi - u}), safeguarded by
      // a bracket F(lo) < r < F(hi) with bisection; starts from "every candidate in M".
      const double u = p.u;
      double ff = 0.0, sl = 0.0, dmn = kInfD, dmx = -kInfD;
#pragma unroll
      for (int c = 0; c < CAP; ++c)
        if (c < pmax && ei[c] >= 0) {
          ff += fmin(fmax(phi_free - d64[c], 0.0), u);
          sl += d64[c];
          dmn = fmin(dmn, d64[c]);
          dmx = fmax(dmx, d64[c]);
        }
      ff = tsum<G>(ff);
      sl = tsum<G>(sl);
      dmn = tmin<G>(dmn);
      dmx = tmax<G>(dmx);
      // free only inside the window (beyond it, the K smallest are capped: F >= K u >= r)
      const bool free = ff <= r && phi_free <= dmx + u;
      double lo = dmn, hi = dmx + u;  // F(lo) = 0 < r <= u T <= F(hi)
      double ph = free ? phi_free : fmin(fmax((r + sl) / (double)max(T, 1), lo), hi);
      bool fin = !active || free || T == 0;
      for (int it = 0; it < 64 && __any_sync(kFull, !fin); ++it) {
        double sM = 0.0;
        int nM = 0, nC = 0;
#pragma unroll
        for (int c = 0; c < CAP; ++c)
          if (c < pmax) {
            const bool lt = d64[c] < ph;
            const bool cp = d64[c] <= ph - u;
            nM += tcount<G>(lt && !cp, gmask);
            nC += tcount<G>(lt && cp, gmask);
            if (lt && !cp) sM += d64[c];
          }
        sM = tsum<G>(sM);
        if (!fin) {
          const double uC = nC > 0 ? u * nC : 0.0;
          const double F = uC + (nM > 0 ? ph * nM - sM : 0.0);
          if (F == r) {
            fin = true;
          } else {
            if (F > r) hi = ph;
            else lo = ph;
            double np = nM > 0 ? (r - uC + sM) / nM : 0.5 * (lo + hi);
            if (!(np > lo && np < hi)) np = 0.5 * (lo + hi);
            if (np == ph || !(hi - lo > 4e-16 * fmax(fabs(hi), fabs(lo)))) fin = true;
            ph = np;
          }
        }
      }
      if (active) {
#pragma unroll
        for (int c = 0; c < CAP; ++c)
          if (c < pmax && ei[c] >= 0) {
            const double x = fmin(fmax(ph - d64[c], 0.0), u);
            if (x > 0.0) emit_smem(C, sd, sc, sa, cap, ei[c], x, vs, b, ei[c] - start);
          }
      }
      __syncwarp();
      continue;
    }
    // Michelot in fp64 on the candidates for the root phi* of F(phi) = sum max(phi - d, 0) = r
    // (every active entry is a candidate and phi* <= r + slack/gamma_i, so F over the candidates
    // is F over the block there): start from all T candidates, phi = (r + sum_S d)/|S|,
    // S = {d < phi}, until |S| is stable (1/|S| from a shared table, within 1 ulp).  The threshold
    // is min(phi_free, phi*): theta = 0 exactly when phi_free <= phi* (F(phi_free) <= r).
    double phi = 0.0;
    bool done = !active || T <= 1;
    {
      double sl = 0.0;
#pragma unroll
      for (int c = 0; c < CAP; ++c)
        if (c < pmax && ei[c] >= 0) sl += d64[c];
      const double sm = tsum<G>(sl);
      if (!done) phi = (r + sm) * (T <= kRcpN ? rcp_s[T] : 1.0 / T);
    }
    int cprev = T;
    for (int it = 0; it < 32 && __any_sync(kFull, !done); ++it) {
      int cnt = 0;
      double sl = 0.0;
#pragma unroll
      for (int c = 0; c < CAP; ++c)
        if (c < pmax) {
          const bool in = d64[c] < phi;
          if constexpr (G <= 4) cnt += in;  // narrow groups: lane counts, one group sum below
          else cnt += tcount<G>(in, gmask);
          if (in) sl += d64[c];
        }
      if constexpr (G <= 4) cnt = tsum<G>(cnt);
      const double sm = tsum<G>(sl);
      if (!done) {
        if (cnt == cprev || cnt == 0) {
          done = true;
        } else {
          cprev = cnt;
          phi = (r + sm) * (cnt <= kRcpN ? rcp_s[cnt] : 1.0 / cnt);
        }
      }
    }
    if (active) {
      const double ph = T == 1 ? phi_free : fmin(phi_free, phi);
      const double cap_x = T == 1 ? r : kInfD;
#pragma unroll
      for (int c = 0; c < CAP; ++c) {
        if (c < pmax && ei[c] >= 0) {
          const double x = fmin(fmax(ph - d64[c], 0.0), cap_x);
          if (x > 0.0) emit_smem(C, sd, sc, sa, cap, ei[c], x, vs, b, ei[c] - start);
        }
      }
    }
    __syncwarp();  // the candidate list is rewritten by the next round
  }
}

// ---------------------------------------------------------------- phase 2: short simplex blocks
// Exact projection onto {x >= 0, sum x <= r} (Eq. 4-5) of every block of a tile.
//
// A warp works a tile of short blocks in rounds of NG = 32/G blocks, G = 2^LG lanes per block:
//  1. fp32 pass: s32 = fl(c + sum_k a_k lambda_k) for every slot, block minimum ref.  Buckets
//     t <= 3 (<= 7 entries): one lane per block, E slots of consecutive entries; t = 4: two lanes,
//     slot k of lane q = entry q + 2k.  Buckets 5..8
//     (stored padded to 4 entries): G = 2^(t-4) lanes, each reading four 4-entry groups with
//     128-bit loads (slot k of lane q = entry 4 (q + (k/4) G) + k%4);
//  2. window: only entries with s - s_min < gamma_i r can be positive (x_j > 0 needs d_j < phi* <=
//     r + d_min); the fp32 filter s32 <= ref + gamma_i r (1 + 1e-6) + slack keeps all of them
//     (slack bounds the fp32 rounding, R7/R14);
//  3. the window's candidates are rescored exactly in fp64, d = (c + sum a lambda - ref)/gamma_i,
//     and the threshold phi* of F(phi) = sum max(phi - d, 0) = r is found by Michelot's iteration
//     (phi = (r + sum_S d)/|S| over S = {d < phi}, from S = all candidates, until |S| is stable):
//     one lane per block works on its own candidates (no shuffles); wider groups compact their
//     candidates so that lane q owns candidates q, q + G, .. (<= CAP) and sum over the group
//     with butterflies -- every group of the round iterates at once;
//  4. threshold min(phi_free, phi*) (theta = 0 exactly when the clamp alone is feasible),
//     x = max(threshold - d, 0), x > 0 scattered with red.global.add.f64.
//  Blocks with more candidates than the group holds (large gamma) are solved right after their
//  round by the whole warp (fp64 Michelot over the block's window, <= 8 entries per lane).

template <int M, int LM, bool WX>
__device__ __forceinline__ float score32_smem(const Ctx<M, LM, WX>& C, const int32_t* sd, const float* sc,
                                              const float* sa, int cap, int ee) {
  float sv = sc[ee];
  const int j = sd[ee];
#pragma unroll
  for (int f = 0; f < M; ++f) sv = fmaf(sa[f * cap + ee], C.lam(f, j), sv);
  return sv;
}

// The whole warp solves one short block [start, end) of the stage (<= 256 stored entries): window
// filter as in the pass, exact fp64 d of the candidates, fp64 Michelot.
template <int M, int LM, bool WX>
__device__ __forceinline__ void warp_block_simplex(Ctx<M, LM, WX>& C, const int32_t* sd, const float* sc,
                                                   const float* sa, int cap, int start, int end, int b, float ref,
                                                   float thr, double vs, double ginv, int lane, const double* rcp_s) {
  double d64[8];
  uint32_t vm = 0;
  const double refd = (double)ref;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int e = start + lane + 32 * c;
    const bool ok = e < end && score32_smem(C, sd, sc, sa, cap, e) <= thr;
    d64[c] = ok ? (score_smem(C, sd, sc, sa, cap, e) - refd) * ginv : kInfD;
    if (ok) vm |= 1u << c;
  }
  warp_michelot(d64, vm, C.p.r, -refd * ginv, rcp_s, [&](int c, double x) {
    const int e = start + lane + 32 * c;
    emit_smem(C, sd, sc, sa, cap, e, x, vs, b, e - start);
  });
}

template <int M, int LM, bool WX, int LG, int E, bool V4, int CAP>
__device__ void small_tile_simplex(Ctx<M, LM, WX>& C, const Tile& tl, const char* stage, int lane,
                                   const uint16_t* rel_s, uint16_t* cand_s, const double* rcp_s) {
  constexpr int G = 1 << LG;
  constexpr int NG = 32 >> LG;
  const GradArgs& p = C.p;
  const int cap = p.tile_cap;
  const int32_t* sd = reinterpret_cast<const int32_t*>(stage);
  const float* sc = reinterpret_cast<const float*>(stage) + cap;
  const float* sa = sc + cap;  // family f at sa + f*cap
  const int gi = lane >> LG, q = lane & (G - 1);
  const int nrounds = (tl.nb + NG - 1) / NG;
  const double r = p.r;
  for (int rd = 0; rd < nrounds; ++rd) {
    const int bb = rd * NG + gi;
    const bool active = bb < tl.nb;
    const int b = tl.b0 + bb;
    int start = 0, end = 0;
    if (active) {
      if (tl.rel_off >= 0) {
        start = rel_s[bb];
        end = rel_s[bb + 1];
      } else {
        start = (int)__ldg(p.blk_rel + b);
        end = bb + 1 < tl.nb ? (int)__ldg(p.blk_rel + b + 1) : tl.nnz;
      }
    }
    double vs = 1.0, ginv = C.invgamma;  // gamma_i = gamma v_i^2
    if (p.vsq && active) {
      vs = (double)__ldg(p.vsq + b);
      ginv = C.invgamma * (double)__ldg(p.vinv + b);
    }
    // ---- 1. fp32 pass
    float s32[E];
    float lmin = kInfF, lmag = 0.f;
    if constexpr (V4) {
      // 4-entry groups: lane q reads groups q, q + G, .. (E/4 of them) of the (padded) block with
      // 128-bit loads; padding has c = +inf, a = 0, so its score is +inf without a test
      static_assert(E % 4 == 0, "whole 4-entry groups per lane");
      const int ng = (end - start) >> 2;
#pragma unroll
      for (int jg = 0; jg < E / 4; ++jg) {
        const int g4 = q + jg * G;
        const int ee = start + 4 * g4;
        int4 d4 = make_int4(0, 0, 0, 0);
        float4 c4 = make_float4(kInfF, kInfF, kInfF, kInfF);
        float4 a4[M];
#pragma unroll
        for (int f = 0; f < M; ++f) a4[f] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g4 < ng) {
          d4 = *reinterpret_cast<const int4*>(sd + ee);
          c4 = *reinterpret_cast<const float4*>(sc + ee);
#pragma unroll
          for (int f = 0; f < M; ++f) a4[f] = *reinterpret_cast<const float4*>(sa + f * cap + ee);
        }
        const int jj[4] = {d4.x, d4.y, d4.z, d4.w};
        float sv[4] = {c4.x, c4.y, c4.z, c4.w}, mg[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) mg[c] = fabsf(sv[c]);
#pragma unroll
        for (int f = 0; f < M; ++f) {
          const float av[4] = {a4[f].x, a4[f].y, a4[f].z, a4[f].w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float lv = C.lam(f, jj[c]);
            sv[c] = fmaf(av[c], lv, sv[c]);
            if constexpr (M > 1) mg[c] = fmaf(fabsf(av[c]), fabsf(lv), mg[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          s32[4 * jg + c] = sv[c];
          lmin = fminf(lmin, sv[c]);
          if constexpr (M > 1) lmag = sv[c] < kInfF ? fmaxf(lmag, mg[c]) : lmag;
        }
      }
    } else {  // scalar slots: slot k of lane q = entry start + q + k G
      const int lim = (end - start) - q;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int ee = start + q + k * G;
        const bool in = k * G < lim;
        const int j = in ? sd[ee] : 0;  // reads past the tile stay inside shared memory (tail pad)
        float sv = in ? sc[ee] : kInfF, mg = fabsf(sv);
#pragma unroll
        for (int f = 0; f < M; ++f) {
          const float a_ = in ? sa[f * cap + ee] : 0.f, lv = C.lam(f, j);
          sv = fmaf(a_, lv, sv);
          if constexpr (M > 1) mg = fmaf(fabsf(a_), fabsf(lv), mg);
        }
        s32[k] = sv;
        lmin = fminf(lmin, sv);
        if constexpr (M > 1) lmag = sv < kInfF ? fmaxf(lmag, mg) : lmag;
      }
    }
    const float ref = tmin<G>(lmin);
    // ---- 2. window (fp32 rounding bound of s_j - ref and of the threshold, K1 step 2)
    const float gr = (float)(r * C.gamma * vs);
    const float slack = M == 1 ? 4.7683716e-7f * (fabsf(ref) + gr) : 2.3841858e-7f * (M + 1) * tmax<G>(lmag);
    const float thr = ref + (gr * 1.000001f + slack);
    uint32_t cm = 0;
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (s32[k] <= thr) cm |= 1u << k;
    if (!active) cm = 0;
    // ---- 3. candidates in registers: lane-local (G = 1) or compacted over the group
    const int nc = __popc(cm);
    int excl = 0, T = nc;
    if constexpr (G > 1) {
      int incl = nc;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, o, G);
        if (q >= o) incl += v;
      }
      T = __shfl_sync(kFull, incl, G - 1, G);
      excl = incl - nc;
    }
    const bool over = T > CAP * G;  // group-uniform
    const double refd = (double)ref;
    double d64[CAP];
    int ei[CAP];
    int own = 0;
    if constexpr (G == 1) {
      uint32_t m = over ? 0u : cm;
#pragma unroll
      for (int c = 0; c < CAP; ++c) {
        d64[c] = kInfD;
        ei[c] = 0;
        if (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          ei[c] = start + k;  // G = 1: slot k is entry k
          d64[c] = (score_smem(C, sd, sc, sa, cap, ei[c]) - refd) * ginv;
          ++own;
        }
      }
    } else {
      uint16_t* lst = cand_s + gi * (CAP * G);
      if (!over) {
        uint32_t m = cm;
        int o = excl;
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          lst[o++] = (uint16_t)(start + slot_entry<LG, V4>(q, k));
        }
      }
      __syncwarp();
      own = over ? 0 : (T - q + G - 1) >> LG;  // candidates q, q + G, ... of the group
#pragma unroll
      for (int c = 0; c < CAP; ++c) {
        d64[c] = kInfD;
        ei[c] = 0;
        if (c < own) {
          ei[c] = lst[q + c * G];
          d64[c] = (score_smem(C, sd, sc, sa, cap, ei[c]) - refd) * ginv;
        }
      }
      __syncwarp();  // the list is rewritten by the next round
    }
    // Michelot in fp64 over the group's candidates, every group at once (warp-uniform loop)
    double sl = 0.0;
#pragma unroll
    for (int c = 0; c < CAP; ++c)
      if (c < own) sl += d64[c];
    const int Tg = over ? 0 : T;
    double phi = (r + tsum<G>(sl)) * rcp_s[Tg];
    int cprev = Tg;
    bool done = Tg <= 1;
    for (int it = 0; it < 64 && __any_sync(kFull, !done); ++it) {
      int cnt = 0;
      double s2 = 0.0;
#pragma unroll
      for (int c = 0; c < CAP; ++c)
        if (c < own && d64[c] < phi) {
          ++cnt;
          s2 += d64[c];
        }
      cnt = tsum<G>(cnt);
      if (__all_sync(kFull, done || cnt == cprev || cnt == 0)) break;  // no group needs the new sum
      s2 = tsum<G>(s2);
      if (!done) {
        if (cnt == cprev || cnt == 0) {
          done = true;
        } else {
          cprev = cnt;
          phi = (r + s2) * rcp_s[cnt];
        }
      }
    }
    // ---- 4. threshold and emission
    const double ph = fmin(-refd * ginv, phi);
#pragma unroll
    for (int c = 0; c < CAP; ++c)
      if (c < own) {
        const double x = fmax(ph - d64[c], 0.0);
        if (x > 0.0) emit_smem(C, sd, sc, sa, cap, ei[c], x, vs, b, ei[c] - start);
      }
    // ---- blocks whose candidates overflow the registers: the whole warp, one block at a time
    unsigned big = __ballot_sync(kFull, q == 0 && active && over);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int s0 = __shfl_sync(kFull, start, src), s1 = __shfl_sync(kFull, end, src);
      const int bk = __shfl_sync(kFull, b, src);
      const float rf = __shfl_sync(kFull, ref, src), th = __shfl_sync(kFull, thr, src);
      const double vsb = __shfl_sync(kFull, vs, src), gb = __shfl_sync(kFull, ginv, src);
      warp_block_simplex<M, LM, WX>(C, sd, sc, sa, cap, s0, s1, bk, rf, th, vsb, gb, lane, rcp_s);
    }
  }
}

// Blocks of one entry (bucket 1): the simplex projection of a scalar is x = clip(-s/gamma_i, 0, r)
// (PAPER.md:125-134 with n = 1), formed directly from the exact fp64 score -- no filter, no threshold
// search.  One block per lane, 32 per round.
template <int M, int LM, bool WX>
__device__ __forceinline__ void single_entry_tile_simplex(Ctx<M, LM, WX>& C, const Tile& tl, const char* stage,
                                                          int lane) {
  const GradArgs& p = C.p;
  const int cap = p.tile_cap;
  const int32_t* sd = reinterpret_cast<const int32_t*>(stage);
  const float* sc = reinterpret_cast<const float*>(stage) + cap;
  const float* sa = sc + cap;
  for (int bb = lane; bb < tl.nb; bb += 32) {
    const int b = tl.b0 + bb;
    const int ee = bb;  // one-entry blocks are contiguous in their tile (plan.cpp): block bb is entry bb
    double vs = 1.0, ginv = C.invgamma;  // gamma_i = gamma v_i^2
    if (p.vsq) {
      vs = (double)__ldg(p.vsq + b);
      ginv = C.invgamma * (double)__ldg(p.vinv + b);
    }
    const double x = fmin(fmax(-score_smem(C, sd, sc, sa, cap, ee) * ginv, 0.0), p.r);
    if (x > 0.0) emit_smem(C, sd, sc, sa, cap, ee, x, vs, b, 0);
  }
}

template <int M, int LM, bool WX>
__device__ __forceinline__ void small_dispatch_simplex(Ctx<M, LM, WX>& C, const Tile& tl, const char* stage,
                                                       int lane, const uint16_t* rel_s, uint16_t* cand_s,
                                                       const double* rcp_s) {
  if (wide_groups(C.p.tile_cap) && tl.bucket >= 5) {  // doubled widths (internal.h round_blocks), E = 8
    switch (tl.bucket) {
      case 5: small_tile_simplex<M, LM, WX, 2, 8, true, 2>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
      case 6: small_tile_simplex<M, LM, WX, 3, 8, true, 2>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
      case 7: small_tile_simplex<M, LM, WX, 4, 8, true, 2>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
      default: small_tile_simplex<M, LM, WX, 5, 8, true, 1>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    }
    return;
  }
  switch (tl.bucket) {  // (LG, E, V4, CAP): E 2^LG >= every stored length of bucket t; round_blocks(t) = 32 / 2^LG
    case 1: single_entry_tile_simplex<M, LM, WX>(C, tl, stage, lane); break;
    case 2: small_tile_simplex<M, LM, WX, 0, 3, false, 3>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 3: small_tile_simplex<M, LM, WX, 0, 7, false, 6>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 4: small_tile_simplex<M, LM, WX, 1, 8, false, 4>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 5: small_tile_simplex<M, LM, WX, 1, 16, true, 4>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 6: small_tile_simplex<M, LM, WX, 2, 16, true, 4>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 7: small_tile_simplex<M, LM, WX, 3, 16, true, 2>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    default: small_tile_simplex<M, LM, WX, 4, 16, true, 2>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
  }
}

template <int M, int LM, bool WX, bool GEN>
__device__ __forceinline__ void small_dispatch(Ctx<M, LM, WX>& C, const Tile& tl, const char* stage, int lane,
                                               const uint16_t* rel_s, uint16_t* cand_s, const double* rcp_s) {
  // box-cut / box keep the base widths also for small tiles (the wide mapping's one-slot-per-candidate
  // solve ran 7x slower on configs[3]); a tile then holds fewer blocks than a round, which only idles lanes
  switch (tl.bucket) {  // (LG, E): E 2^LG >= every stored length of bucket t; round_blocks(t) = 32 / 2^LG
    case 1:
    case 2:
    case 3: small_tile<M, LM, WX, 0, 8, GEN>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 4: small_tile<M, LM, WX, 1, 8, GEN>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 5: small_tile<M, LM, WX, 1, 16, GEN>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 6: small_tile<M, LM, WX, 2, 16, GEN>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    case 7: small_tile<M, LM, WX, 3, 16, GEN>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
    default: small_tile<M, LM, WX, 4, 16, GEN>(C, tl, stage, lane, rel_s, cand_s, rcp_s); break;
  }
}

// KIND: DL_PROJ_SIMPLEX / DL_PROJ_BOXCUT / DL_PROJ_BOX; LM: lambda placement (kLam*).
template <int M, int LM, bool WX, int KIND>
__global__ void __launch_bounds__(kThreads, 1) fused_grad_kernel(const __grid_constant__ GradArgs p) {
  extern __shared__ __align__(128) char smem[];
  SmemHead* head = reinterpret_cast<SmemHead*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* trace = p.trace ? p.trace + 5 * blockIdx.x : nullptr;
  if (trace && threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    trace[0] = sm;
    trace[1] = globaltimer();
    trace[4] = 0;  // tile count, added by every warp after the barrier below
  }
  char* after_head = smem + 2048;
  float* lam_s = nullptr;
  size_t lam_bytes = 0;
  if constexpr (LM != kLamGlobal) {  // stage all duals, or those of the hot labels [0, H) per family
    const int H = LM == kLamSmem ? p.J : p.lam_hot;
    lam_s = reinterpret_cast<float*>(after_head);
    lam_bytes = ((size_t)M * H * 4 + 127) / 128 * 128;
    for (int f = 0; f < M; ++f)
      for (int i = threadIdx.x; i < H; i += kThreads) lam_s[f * H + i] = __ldg(p.lam + (size_t)f * p.J + i);
  }
  char* tilebuf = after_head + lam_bytes;
  const uint32_t stage_bytes = (uint32_t)p.tile_cap * (8u + 4u * M);
  if (lane == 0) {
    mbar_init(&head->mbar[warp][0], 1);
    mbar_init(&head->mbar[warp][1], 1);
  }
  for (int i = threadIdx.x; i <= kRcpN; i += kThreads) head->rcp[i] = c_rcp[i];
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[2] = globaltimer();

  const double gamma = p.gamma_ptr ? *p.gamma_ptr : p.gamma_val;
  Ctx<M, LM, WX> C(p, lam_s, gamma);
  unsigned ntiles = 0;  // tiles this warp worked (trace only)

  // ---- phase 1: big blocks, groups of 16 / 8 / 4 / 2 warps; barrier ids unique per group
  for (int ph = 0; ph < kNumBigPhases; ++ph) {
    if (p.ph_begin[ph] == p.ph_begin[ph + 1]) continue;
    BigGroup g;
    g.gw = 16 >> ph;
    g.G = g.gw * 32;
    const int grp = warp / g.gw;
    g.warp0 = grp * g.gw;
    g.gtid = (warp - g.warp0) * 32 + lane;
    g.bar = (1 << ph) + grp;  // phase 0: 1, phase 1: 2-3, phase 2: 4-7, phase 3: 8-15
    g.lane = lane;
    g.warp = warp;
    g.head = head;
    // scratch: this group's warps' tile buffers (doubles), else a global slice
    double* scr_smem = reinterpret_cast<double*>(tilebuf + (size_t)g.warp0 * 2 * stage_bytes);
    const int scr_cap = (int)((size_t)g.gw * 2 * stage_bytes / 8);
    for (;;) {
      if (g.gtid == 0) head->slot[g.bar] = atomicAdd(p.ctr + ph, 1) + p.ph_begin[ph];
      g.sync();
      const int ti = head->slot[g.bar];
      if (ti >= p.ph_begin[ph + 1]) break;
      const Tile tl = p.tiles[ti];
      ntiles += g.gtid == 0;
      double* scr = tl.nnz <= scr_cap ? scr_smem : p.gscratch + (size_t)blockIdx.x * p.gscratch_per_cta;
      if constexpr (KIND == DL_PROJ_SIMPLEX)
        big_block_simplex<M, LM, WX>(C, g, tl, scr_smem, scr_cap, scr);
      else
        big_block<M, LM, WX>(C, g, tl, scr);
    }
  }

  // ---- phase 2: small tiles.  Each warp runs its own asynchronous stream: tiles are claimed
  // in chunks of kChunk (one atomic per chunk, claimed a chunk ahead); the chunk's tile
  // descriptors arrive by a 128-B bulk copy into a shared slot; every tile's dest / c / a_k
  // arrays and its block offsets arrive by bulk copies into a double-buffered stage.  No
  // global load sits on the critical path of a tile.
  {
    constexpr int kChunk = 8;  // tiles per claim (one atomic) and per descriptor bulk copy
    const int s_begin = p.ph_begin[kNumBigPhases], s_end = p.ph_begin[kNumBigPhases + 1];
    char* mybuf = tilebuf + (size_t)warp * 2 * stage_bytes;
    constexpr int kMeta = kMetaBytes;
    char* meta = tilebuf + (size_t)kWarps * 2 * stage_bytes + (size_t)warp * kMeta;
    const Tile* dslot = reinterpret_cast<const Tile*>(meta);                 // [2][kChunk]
    const uint16_t* rslot = reinterpret_cast<const uint16_t*>(meta + 512);   // [2][64]
    uint16_t* cslot = reinterpret_cast<uint16_t*>(meta + 768);  // [128] candidate list
    uint64_t* bars = head->mbar[warp];
    uint64_t* dbars = head->mbar_desc[warp];
    if (lane == 0) {
      mbar_init(&dbars[0], 1);
      mbar_init(&dbars[1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    // lane 0 claims a chunk; the value is broadcast only when it is used (a chunk later), so
    // the atomic's latency is not waited on
    auto grab = [&]() {
      int c = 0;
      if (lane == 0) c = atomicAdd(p.ctr + kNumBigPhases, 1);
      return c;
    };
    auto first_of = [&](int raw) { return s_begin + kChunk * __shfl_sync(kFull, raw, 0); };
    auto issue_desc = [&](int first, int slot) {
      if (lane == 0 && first < s_end) {
        fence_proxy_async();
        mbar_expect_tx(&dbars[slot], kChunk * (uint32_t)sizeof(Tile));
        tma_bulk_g2s(meta + slot * kChunk * sizeof(Tile), p.tiles + first, kChunk * (uint32_t)sizeof(Tile),
                     &dbars[slot]);
      }
    };
    auto issue_tile = [&](const Tile& t, int st) {
      if (lane == 0) {
        const uint32_t n4 = (uint32_t)((t.nnz + kAlign - 1) / kAlign * kAlign);
        const uint32_t bytes = n4 * 4u;
        const uint32_t rbytes = t.rel_off >= 0 ? (uint32_t)((2 * (t.nb + 1) + 15) & ~15) : 0u;
        char* dst = mybuf + (size_t)st * stage_bytes;
        fence_proxy_async();
        mbar_expect_tx(&bars[st], bytes * (2u + M) + rbytes);
        const uint64_t pol = evict_first_policy();
        tma_bulk_g2s_stream(dst, p.dest + t.off, bytes, &bars[st], pol);
        tma_bulk_g2s_stream(dst + (size_t)p.tile_cap * 4, p.c + t.off, bytes, &bars[st], pol);
#pragma unroll
        for (int f = 0; f < M; ++f)
          tma_bulk_g2s_stream(dst + (size_t)p.tile_cap * (8 + 4 * f), p.a + f * p.a_stride + t.off, bytes, &bars[st],
                              pol);
        if (rbytes) tma_bulk_g2s(meta + 512 + st * 128, p.rel_pool + t.rel_off, rbytes, &bars[st]);
      }
    };
    uint32_t phase = 0u, dphase = 0u;  // mbarrier parities, bit s for slot s (kept in registers)
    int c0 = first_of(grab()), c1 = first_of(grab());
    int ds = 0;  // descriptor slot of chunk c0
    issue_desc(c0, 0);
    issue_desc(c1, 1);
    int c2raw = grab();
    int pos = 0, st = 0;
    Tile t{};
    bool have = c0 < s_end;
    if (have) {
      mbar_wait(&dbars[0], dphase & 1u);
      dphase ^= 1u;
      t = dslot[0];
      issue_tile(t, 0);
    }
    while (have) {
      // descriptor of the next tile: same chunk, or the first of the next chunk
      Tile tn{};
      bool nhave;
      const bool same = pos + 1 < kChunk && c0 + pos + 1 < s_end;
      if (same) {
        tn = dslot[ds * kChunk + pos + 1];
        nhave = true;
      } else {
        nhave = c1 < s_end;
        if (nhave) {
          mbar_wait(&dbars[ds ^ 1], (dphase >> (ds ^ 1)) & 1u);
          dphase ^= 1u << (ds ^ 1);
          tn = dslot[(ds ^ 1) * kChunk];
        }
      }
      if (nhave) issue_tile(tn, st ^ 1);
      mbar_wait(&bars[st], (phase >> st) & 1u);
      phase ^= 1u << st;
      if constexpr (KIND == DL_PROJ_SIMPLEX)
        small_dispatch_simplex<M, LM, WX>(C, t, mybuf + (size_t)st * stage_bytes, lane, rslot + st * 64, cslot,
                                          head->rcp);
      else
        small_dispatch<M, LM, WX, true>(C, t, mybuf + (size_t)st * stage_bytes, lane, rslot + st * 64, cslot,
                                        head->rcp);
      __syncwarp();
      ++ntiles;
      if (same) {
        ++pos;
      } else {  // chunk c0 done: its descriptor slot takes chunk c2
        if (trace && lane == 0) p.trace[5 * gridDim.x + (c0 - s_begin) / kChunk] = globaltimer();
        const int c2 = first_of(c2raw);
        __syncwarp();
        issue_desc(c2, ds);
        c0 = c1;
        c1 = c2;
        ds ^= 1;
        pos = 0;
        c2raw = c1 < s_end ? grab() : (s_end - s_begin) / kChunk + 1;  // past the end
      }
      t = tn;
      have = nhave;
      st ^= 1;
    }
  }

  // ---- objective scalars: warp reduce, one fp64 atomic per warp
  double cx = C.cx, rg = C.reg;
  float nx = C.nx;
  for (int o = 16; o > 0; o >>= 1) {
    cx += __shfl_xor_sync(kFull, cx, o);
    rg += __shfl_xor_sync(kFull, rg, o);
    nx += __shfl_xor_sync(kFull, nx, o);
  }
  if (lane == 0) {
    const size_t n = (size_t)M * p.J;
    atomicAdd(C.acc + n + 0, cx);
    atomicAdd(C.acc + n + 1, rg);
    atomicAdd(C.acc + n + 2, (double)nx);
    if (trace) atomicAdd(trace + 4, (unsigned long long)ntiles);
  }
  if (trace) {
    __syncthreads();
    if (threadIdx.x == 0) trace[3] = globaltimer();
  }
}

template <int M, int LM, bool WX, int KIND>
cudaError_t launch_t(const GradArgs& a, int ctas, size_t smem, cudaStream_t s) {
  auto k = fused_grad_kernel<M, LM, WX, KIND>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<ctas, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int M, int KIND>
cudaError_t launch_k(const GradArgs& a, int ctas, size_t smem, cudaStream_t s) {
  const bool wx = a.x_out != nullptr;
  if (a.lam_mode == kLamSmem)
    return wx ? launch_t<M, kLamSmem, true, KIND>(a, ctas, smem, s) : launch_t<M, kLamSmem, false, KIND>(a, ctas, smem, s);
  // kLamHot, and kLamGlobal as its special case lam_hot = 0 (every label read from global memory)
  GradArgs b = a;
  if (a.lam_mode != kLamHot) b.lam_hot = 0;
  return wx ? launch_t<M, kLamHot, true, KIND>(b, ctas, smem, s) : launch_t<M, kLamHot, false, KIND>(b, ctas, smem, s);
}

}  // namespace

// one translation unit per (family count, polytope kind): grad_m<M>_k<KIND>.cu, compiled in parallel
template <>
cudaError_t launch_fused_grad_mk<DL_GRAD_M, DL_GRAD_KIND>(const GradArgs& a, int ctas, size_t smem, cudaStream_t s) {
  return launch_k<DL_GRAD_M, DL_GRAD_KIND>(a, ctas, smem, s);
}

}  // namespace dl
