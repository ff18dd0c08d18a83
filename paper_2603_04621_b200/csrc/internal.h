// Internal declarations shared by the host planner, the kernels and the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "dualip.h"

#ifdef __CUDACC__
#include <cuda_runtime.h>
#else
typedef struct CUstream_st* cudaStream_t;
typedef struct CUgraphExec_st* cudaGraphExec_t;
#endif

namespace dl {

// ---- layout (mirrors oracle/layout.py) -------------
constexpr int kBigBucket = 9;      // buckets >= 9 (len >= 256): multi-warp groups
constexpr int kAlign = 4;          // entries: 16-byte TMA alignment of every tile
constexpr int kWarps = 16;         // warps per CTA of the fused kernel
constexpr int kThreads = kWarps * 32;
constexpr int kNumBigPhases = 4;   // group widths 16, 8, 4, 2 warps
constexpr int kRelMax = 63;        // tiles with fewer blocks stream their block offsets with the data
// per-warp metadata in shared memory: 2 descriptor-chunk slots (2 x 8 tiles x 32 B) + 2 block-offset
// slots (2 x 128 B) + the round's compacted candidate list (128 x u16)
constexpr int kMetaBytes = 1024;
inline int meta_bytes(int) { return kMetaBytes; }

struct alignas(16) Tile {
  int64_t off;     // first entry (multiple of kAlign)
  int32_t nnz;     // entries of the tile (sum of its block lengths)
  int32_t b0;      // first block (layout order)
  int32_t nb;      // blocks in the tile
  int32_t bucket;  // t = floor(log2 len) + 1 of its blocks
  int32_t rel_off; // start (uint16 units, multiple of 8) of the tile's block offsets in rel_pool, or -1
  int32_t pad1;
};
static_assert(sizeof(Tile) == 32, "tile descriptor is 32 bytes");

struct Plan {
  std::vector<int64_t> perm;     // source of each block
  std::vector<int64_t> blk_off;  // entry offset of each block
  std::vector<Tile> tiles;
  int64_t total = 0;             // entries incl. alignment gaps
  int32_t max_len = 0;
  int32_t num_buckets = 0;
  int32_t ph_begin[kNumBigPhases + 2] = {0, 0, 0, 0, 0, 0};  // tile ranges: 4 big phases + small
};

inline int bucket_of(int64_t s) { return 64 - __builtin_clzll((unsigned long long)s); }
// buckets [kPadBucket, kBigBucket) (16..255 entries) store every block padded to a multiple of
// kAlign entries (padding: label 0, c = +inf, a = 0) so that the fused kernel reads them 4 entries
// per 128-bit shared-memory load
constexpr int kPadBucket = 5;
inline int64_t stored_len(int64_t s) {
  const int t = bucket_of(s);
  return (t >= kPadBucket && t < kBigBucket) ? (s + kAlign - 1) / kAlign * kAlign : s;
}
// blocks of a small bucket one warp works per round: 32 / G, G the group width of the fused
// kernel (1 lane for t <= 3, 2 for t = 4, 2^(t-4) for t = 5..8 -- doubled for tiles below
// kWideCap entries, so that a round of blocks of the bucket's typical length fits one tile)
constexpr int kWideCap = 384;
#ifdef __CUDACC__
__host__ __device__
#endif
inline bool wide_groups(int tile_cap) { return tile_cap < kWideCap; }
inline int round_blocks(int bucket, int tile_cap) {
  if (bucket <= 3) return 32;
  if (bucket == 4) return 16;
  return 32 >> (bucket - (wide_groups(tile_cap) ? 3 : 4));
}
inline int big_phase_of(int bucket) {  // bucket >= 12 -> phase 0 (16 warps) ... 9 -> phase 3 (2 warps)
  return bucket >= 12 ? 0 : 12 - bucket;
}

Plan make_plan(const int64_t* row_ptr, int64_t num_sources, int32_t tile_cap);
// lambda placement of the fused kernel: kLamGlobal -> every dual read
// from global memory (L2); kLamSmem -> all m*J duals staged in shared memory; kLamHot -> the
// duals of destination labels [0, hot) staged (labels = popularity order, R15), the rest global
enum { kLamGlobal = 0, kLamSmem = 1, kLamHot = 2 };
struct SmemRule {
  int32_t tile_cap;
  int32_t lam_mode;
  int32_t hot;  // labels cached per family (J for kLamSmem)
};
SmemRule smem_rule(int32_t m, int32_t J, int32_t kind);
size_t fused_smem_bytes(int32_t m, int32_t kind, int32_t tile_cap, int32_t hot);
int32_t tile_cap_rule(int32_t m, int32_t J, int* lambda_in_smem);  // = smem_rule(m, J, simplex)

void set_error(const std::string& msg);

// ---- device-side AGD state ------------------------------------------------
struct AgdDev {
  double gamma;       // gamma_t used by the next evaluation
  double gamma_prev;  // gamma_{t-1}
  double eta;         // last step
  int64_t t;          // next iteration index
  int64_t k;          // momentum counter
  double gamma0, gamma_min, gamma_ref, max_step, init_step;
  int32_t halve_every, continuation;
  int64_t hist_cap;
};

// ---- kernel launch interfaces (implemented in grad.cu / step.cu) ----------
struct GradArgs {
  const int32_t* dest;
  const float* c;
  const float* a;
  int64_t a_stride;
  const Tile* tiles;
  int32_t ph_begin[kNumBigPhases + 2];
  const uint16_t* blk_rel;
  const uint16_t* rel_pool; // per small tile with < kRelMax blocks: 16-B aligned {rel_0..rel_{nb-1}, nnz}
  const float* vsq;        // per block v_i^2, or nullptr
  const float* vinv;       // per block 1/v_i^2 (with vsq)
  const int64_t* orig_off; // per block original CSR offset (primal output)
  const float* lam;        // [m*J] fp32 duals, indexed by destination LABEL (k*J + label)
  int32_t J, m;
  int32_t lam_mode;        // kLamGlobal / kLamSmem / kLamHot
  int32_t lam_hot;         // labels [0, lam_hot) staged in shared memory (kLamHot; J for kLamSmem)
  const double* gamma_ptr; // device gamma (solver) or nullptr -> gamma_val
  double gamma_val;
  double r, u;             // polytope caps (inf where absent)
  int32_t kind;
  int32_t tile_cap;
  double* acc;             // per-CTA partial accumulators: copy (blockIdx % acc_copies) at acc + copy * acc_stride,
                           // rows [m*J + 4] by label (summed by launch_partial_sum)
  int64_t acc_stride;
  int32_t acc_copies;
  int32_t num_sms;         // SM count (SM id -> accumulator copy when copies < CTAs)
  int32_t* ctr;            // [8] work-queue counters (zeroed before launch)
  float* x_out;            // primal output (original order) or nullptr
  double* gscratch;        // global fp64 d-scratch for blocks beyond the smem scratch
  int64_t gscratch_per_cta;
  unsigned long long* trace;  // per CTA {smid, t_start, t_staged, t_end, tiles} (dl_debug_trace) or nullptr
};

cudaError_t launch_fused_grad(const GradArgs& a, int ctas, size_t smem, cudaStream_t s);
template <int M, int KIND>
cudaError_t launch_fused_grad_mk(const GradArgs& a, int ctas, size_t smem, cudaStream_t s);

constexpr int kStepCtas = 64;  // CTAs of the AGD reduce kernel (partials buffer 5 x kStepCtas)

struct StepArgs {
  int32_t n;               // m*J
  const double* D;         // Jacobi diagonal
  const float* b;
  double* acc;             // [n+4], zeroed on exit
  int32_t* ctr;            // zeroed on exit
  double *lam1, *lam2, *lam2_prev, *G_prev;
  float* mu;
  AgdDev* st;
  dl_iter_record* hist;
  double* part;            // [5 * kStepCtas] per-CTA partial sums
  int32_t* done;           // CTA completion counter (0 between steps)
  double* scal;            // [2] eta, beta of the step
};
cudaError_t launch_agd_step(const StepArgs& a, cudaStream_t s);
// acc[r] = sum over copies c (in order) of part[c * stride + r] for r < n, and part[c * stride + r] = 0
// (the per-CTA partials of the fused pass -> the accumulator; deterministic order)
cudaError_t launch_partial_sum(double* part, int64_t stride, int32_t copies, int64_t n, double* acc, cudaStream_t s);

struct FinalizeArgs {
  int32_t n, J;
  const double* acc;       // label order
  const float* b;          // label order
  const float* lam;        // label order
  const int32_t* lab;      // destination -> label
  double* grad;            // ORIGINAL order
  double* obj;
  int32_t partial;
};
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t s);

// row norms over the layout (dest = labels) written in ORIGINAL order via unlab
cudaError_t launch_row_sqnorms(const int32_t* dest, const float* a, int64_t a_stride, int64_t n_entries, int32_t m,
                               int32_t J, const int32_t* unlab, double* out, cudaStream_t s);
// D[k*J + lab[j]] = 1/sqrt(rowsq[k*J + j]) (rowsq ORIGINAL order; NULL -> 1)
cudaError_t launch_jacobi_diag(const double* rowsq, const int32_t* lab, double* D, int32_t m, int32_t J,
                               cudaStream_t s);
cudaError_t launch_fill_f64(double* p, double v, int64_t n, cudaStream_t s);
// out[k*J + j] = D[k*J + lab[j]] * lam[k*J + lab[j]]  (label order -> ORIGINAL order)
cudaError_t launch_scale_out(const double* D, const double* lam, const int32_t* lab, double* out, int32_t m,
                             int32_t J, cudaStream_t s);
// out[k*J + lab[j]] = in[k*J + j] (f32: ORIGINAL -> label order), and the inverse gather
cudaError_t launch_permute_f32(const float* in, const int32_t* lab, float* out, int32_t m, int32_t J, int inverse,
                               cudaStream_t s);
// relabel an fp64 / fp32 label-ordered vector from labels lab_old to lab_new (via unlab_old)
cudaError_t launch_relabel_vec_f64(double* v, double* tmp, const int32_t* unlab_old, const int32_t* lab_new,
                                   int32_t m, int32_t J, cudaStream_t s);
cudaError_t launch_relabel_vec_f32(float* v, float* tmp, const int32_t* unlab_old, const int32_t* lab_new, int32_t m,
                                   int32_t J, cudaStream_t s);
// dest[e] = lab_new[unlab_old[dest[e]]] over the layout
cudaError_t launch_relabel_dest(int32_t* dest, int64_t n, const int32_t* unlab_old, const int32_t* lab_new,
                                cudaStream_t s);
// counts[j] += #edges with dest j (int64), over a raw (original-index) dest array
cudaError_t launch_dest_histogram(const int32_t* dest, int64_t n, int32_t J, unsigned long long* counts,
                                  cudaStream_t s);

// Scatter of the caller's CSR sources [i0, i1) into the layout.  The input arrays hold the
// entries [e0, e0 + n_in) of the CSR (a chunk: a[k * a_in_stride + e - e0]); row_ptr is the full
// device copy; v (if given) is indexed by source - i0.
struct LayoutArgs {
  const int64_t* row_ptr;
  const int32_t* dest;
  const float* a;
  const float* c;
  const float* v;
  int64_t i0, i1, e0, a_in_stride, a_stride_out;
  int32_t m;
  const int32_t* blk_of_src;  // block of each source (-1: empty)
  const int64_t* blk_off;
  const int32_t* lab;         // destination -> label
  int32_t* dest_out;
  float* c_out;
  float* a_out;
  float* vsq_out;
  float* vinv_out;
  int32_t J;
  int32_t* bad;  // set to 1 if a dest index is outside [0, J)
};
cudaError_t launch_build_layout(const LayoutArgs& a, cudaStream_t s);

}  // namespace dl
