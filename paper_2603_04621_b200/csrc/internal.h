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
constexpr int kMetaBytes = 768;    // per warp: 2 descriptor-chunk slots (128 B) + 2 rel slots (128 B) + candidate list (256 B)

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
// blocks of a small bucket one warp works per round: 32 / G, G the group width of the fused
// kernel (small_dispatch: 1 lane for t <= 3, then 2, 4, 4, 8, 16 lanes for t = 4..8)
inline int round_blocks(int bucket) {
  return bucket <= 3 ? 32 : bucket == 4 ? 16 : bucket <= 6 ? 8 : bucket == 7 ? 4 : 2;
}
inline int big_phase_of(int bucket) {  // bucket >= 12 -> phase 0 (16 warps) ... 9 -> phase 3 (2 warps)
  return bucket >= 12 ? 0 : 12 - bucket;
}

Plan make_plan(const int64_t* row_ptr, int64_t num_sources, int32_t tile_cap);
int32_t tile_cap_rule(int32_t m, int32_t J, int* lambda_in_smem);
size_t fused_smem_bytes(int32_t m, int32_t J, int32_t tile_cap, int lambda_in_smem);

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
struct DeferEntry {  // a short simplex block handed from the fused kernel to deferred_kernel
  int64_t off;       // first entry in the permuted arrays
  int32_t b;         // block (layout order)
  int32_t len;
};

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
  const float* lam;        // [m*J]
  int32_t J, m;
  const double* gamma_ptr; // device gamma (solver) or nullptr -> gamma_val
  double gamma_val;
  double r, u;             // polytope caps (inf where absent)
  int32_t kind;
  int32_t tile_cap;
  int32_t lam_smem;
  double* acc;             // [m*J + 4]
  int32_t* ctr;            // [8] work-queue counters (zeroed before launch); [6] = deferred blocks
  DeferEntry* defer;       // deferred-block queue (simplex / box kinds)
  int32_t defer_cap;
  float* x_out;            // primal output (original order) or nullptr
  double* gscratch;        // global fp64 d-scratch for blocks beyond the smem scratch
  int64_t gscratch_per_cta;
};

cudaError_t launch_fused_grad(const GradArgs& a, int ctas, size_t smem, cudaStream_t s);
template <int M>
cudaError_t launch_fused_grad_m(const GradArgs& a, int ctas, size_t smem, cudaStream_t s);

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

struct FinalizeArgs {
  int32_t n;
  const double* acc;
  const float* b;
  const float* lam;
  double* grad;
  double* obj;
  int32_t partial;
};
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t s);

cudaError_t launch_row_sqnorms(const int32_t* dest, const float* a, int64_t a_stride, int64_t n_entries, int32_t m,
                               int32_t J, double* out, cudaStream_t s);
cudaError_t launch_jacobi_diag(const double* rowsq, double* D, int32_t n, cudaStream_t s);
cudaError_t launch_fill_f64(double* p, double v, int64_t n, cudaStream_t s);
cudaError_t launch_scale_out(const double* D, const double* lam, double* out, int32_t n, cudaStream_t s);

struct LayoutArgs {
  const int64_t* row_ptr;
  const int32_t* dest;
  const float* a;
  const float* c;
  const float* v;
  int64_t nnz, a_stride_out;
  int32_t m;
  int64_t num_blocks;
  const int64_t* perm;
  const int64_t* blk_off;
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
