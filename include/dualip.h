/*
 * dualip.h — C ABI of the B200-native dual-gradient hot path for ridge-regularised
 * dual ascent on matching LPs (arXiv 2603.04621, "PAPER.md" below).
 *
 * The LP (Eq. 1):  min c^T x  s.t.  A x <= b,  x in C.
 * Matching structure (Definition 1): the m*J complex rows
 * (family k, destination j) touch variable x_ij of source i through the diagonal
 * coefficient a_kij; C is a product of per-source polytopes.
 * Ridge-regularised dual (Eq. 2):
 *     g(lambda) = min_{x in C} c^T x + (gamma/2) x^T D_v^2 x + lambda^T (A x - b)
 *     grad g(lambda) = A x*(lambda) - b,  x*_i = Pi_{C_i}(-(c_i + A_i^T lambda) / (gamma v_i^2)).
 *
 * Conventions for every call
 *  - All array arguments are plain pointers.  "device" = CUDA device memory on the
 *    problem's device (any allocator); "host" = host memory (pinned recommended).
 *  - Nothing is retained from caller buffers after a call returns: the problem
 *    copies what it needs into memory it owns (released by dl_problem_destroy).
 *  - Calls are asynchronous on the problem's stream unless stated otherwise;
 *    device outputs are valid once that stream has been synchronised.
 *  - Errors: every call returns dl_status; DL_OK = 0.  On error the problem is
 *    left unchanged where possible and dl_last_error() gives a message
 *    (thread-local, valid until the next failing call on that thread).
 *  - Not thread-safe per problem: serialise calls on one dl_problem.
 *  - There is no CPU fallback: a call that cannot run on the GPU fails.
 */
#ifndef DUALIP_H
#define DUALIP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DL_ABI_VERSION 3

typedef enum {
  DL_OK = 0,
  DL_ERR_INVALID = 1,     /* bad argument / inconsistent sizes                     */
  DL_ERR_CUDA = 2,        /* CUDA runtime error (message has the CUDA string)      */
  DL_ERR_OOM = 3,         /* device or host allocation failed                      */
  DL_ERR_STATE = 4,       /* call out of order (e.g. dl_dual_step before agd_init) */
  DL_ERR_NCCL = 5,        /* NCCL missing or failed                                 */
  DL_ERR_UNSUPPORTED = 6  /* configuration outside what this build supports         */
} dl_status;

/* Simple-constraint polytopes C_i (R1). */
typedef enum {
  DL_PROJ_SIMPLEX = 0,  /* {x >= 0, sum_j x_ij <= r}         (Eq. 4-5, r = 1 in the paper) */
  DL_PROJ_BOXCUT = 1,   /* {0 <= x <= u, sum_j x_ij <= r}    ("box-cut", sum <= k)          */
  DL_PROJ_BOX = 2       /* {0 <= x <= u}                                                      */
} dl_proj_kind;

typedef struct dl_problem dl_problem; /* opaque, owns device memory */

/* One matching LP (or one rank's shard of sources) in source-major CSR.
 * one column of the sparse tensor per source i holding diag(D_i). */
typedef struct {
  int64_t num_sources;    /* I  (sources of this shard), >= 0                          */
  int32_t num_dests;      /* J  >= 1                                                   */
  int32_t num_families;   /* m  in [1, 4] (constraint families, Definition 1)          */
  int64_t nnz;            /* stored edges = row_ptr[I]                                 */
  const int64_t* row_ptr; /* device [I+1], row_ptr[0] = 0, nondecreasing               */
  const int32_t* dest;    /* device [nnz], j in [0,J), strictly ascending per source   */
  const float* a;         /* device [m*nnz], family-major: a[k*nnz + e] = a_kij        */
  const float* c;         /* device [nnz], objective coefficient c_ij (minimisation)  */
  const float* b;         /* device [m*J], family-major right-hand side b[k*J + j]     */
  const float* v;         /* device [I] per-source primal scale v_i > 0 (PAPER.md:299-330,
                             DESIGN.md R4: block i regularised by gamma*v_i^2), or NULL */
  int32_t proj_kind;      /* dl_proj_kind                                              */
  double proj_r;          /* sum cap r > 0 (simplex, box-cut); ignored for box         */
  double proj_u;          /* coordinate cap u > 0 (box-cut, box); ignored for simplex  */
  int32_t device;         /* CUDA device ordinal                                       */
  void* stream;           /* cudaStream_t for all work on this problem (NULL: a new
                             non-blocking stream owned by the problem)                 */
} dl_problem_desc;

typedef struct {
  int64_t num_sources, nnz;
  int64_t nnz_layout;     /* entries of the permuted arrays incl. 16-B alignment gaps */
  int64_t num_blocks;     /* nonempty source blocks                                    */
  int64_t num_tiles, num_big_tiles;
  int32_t num_dests, num_families;
  int32_t tile_cap;       /* max entries of a small tile (layout parameter)            */
  int32_t lambda_in_smem; /* 1 if lambda is staged in shared memory                    */
  int32_t max_block_len, num_buckets;
  int32_t num_sms, ctas;  /* grid of the fused kernel                                  */
  int64_t device_bytes;   /* device memory owned by the problem                        */
  int32_t has_comm;       /* 1 once dl_comm_init created an NCCL communicator (any world) */
  int32_t comm_rank, comm_world;
  int32_t relabeled;      /* 1 if destinations are relabeled by popularity (R15) */
  int32_t lambda_hot;     /* destination labels [0, lambda_hot) whose duals sit in shared memory
                             (= num_dests when all of lambda fits; 0 when none is cached)     */
  int32_t pad_;
} dl_problem_info;

/* ---- version / errors ---------------------------------------------------- */
int dl_abi_version(void);
const char* dl_last_error(void);

/* ---- A1: problem + layout ----------------------------- */
/* Copies the CSR into the bucket-permuted, tile-aligned layout of DESIGN.md
 * "HBM layout".  Synchronises the stream once (reads row_ptr to plan). */
dl_status dl_problem_create(const dl_problem_desc* desc, dl_problem** out);
/* Same, but row_ptr, dest, a, c, b and v are HOST pointers (any host memory).  The edge
 * arrays are streamed to the device in source chunks straight into the layout, so the
 * device never holds a second copy of the input (BASELINE configs[2]: 5e9 edges).
 * Synchronous. */
dl_status dl_problem_create_host(const dl_problem_desc* desc, dl_problem** out);
dl_status dl_problem_destroy(dl_problem* p);
dl_status dl_problem_get_info(const dl_problem* p, dl_problem_info* out);
/* Copies the layout back to HOST buffers (synchronous):
 *   perm[num_blocks]    source id of each block in layout order
 *   blk_off[num_blocks] entry offset of each block in the permuted arrays
 *   tiles[5*num_tiles]  (first_block, num_blocks, entry_offset, num_entries, bucket)
 * Any pointer may be NULL to skip it. */
dl_status dl_problem_layout(const dl_problem* p, int64_t* perm, int64_t* blk_off, int64_t* tiles);
/* Copies the permuted DEVICE arrays back to HOST (synchronous, tests):
 * dest[nnz_layout], c[nnz_layout], a[m*nnz_layout]; NULL skips. */
dl_status dl_problem_layout_data(const dl_problem* p, int32_t* dest, float* c, float* a);

/* Destination labels (R15): lab[j] = label of destination j (a permutation of
 * [0, J)).  Labels order destinations by edge count, descending (ties: j ascending), when
 * lambda does not fit in shared memory, so that the duals of the most-gathered destinations
 * are the ones cached on chip; identity otherwise.  HOST output [num_dests]. */
dl_status dl_problem_dest_labels(const dl_problem* p, int32_t* lab);

/* Host-only planners (no GPU needed; same code dl_problem_create uses).
 * dl_plan_tiles: call with NULL outputs to get the counts, then with buffers
 * perm[num_blocks], blk_off[num_blocks], tiles[5*num_tiles]. row_ptr is HOST. */
dl_status dl_plan_tiles(const int64_t* row_ptr, int64_t num_sources, int32_t tile_cap, int64_t* perm,
                        int64_t* blk_off, int64_t* tiles, int64_t* num_blocks, int64_t* num_tiles,
                        int64_t* total_entries);
/* Balanced contiguous source split for `world` ranks:
 * bounds[w] = min{i : row_ptr[i] >= floor(w*nnz/world)}, bounds[0]=0, bounds[world]=I. */
dl_status dl_plan_shards(const int64_t* row_ptr, int64_t num_sources, int32_t world, int64_t* bounds);
/* The tile capacity rule used by dl_problem_create for (m, J). */
int32_t dl_tile_cap(int32_t num_families, int32_t num_dests);

/* ---- A2: Jacobi row normalisation --------------------- */
/* out[m*J] (device, fp64) = ||A_r*||_2^2 over THIS shard's edges (sum over shards
 * = the global row norms; all-reduce them before dl_set_jacobi when sharded). */
dl_status dl_row_sqnorms(dl_problem* p, double* out);
/* D_rr = 1/sqrt(row_sqnorm[r]) (1 on zero rows) used by the AGD state (R3).
 * row_sqnorm: device [m*J] fp64, GLOBAL norms.  NULL resets D = I. */
dl_status dl_set_jacobi(dl_problem* p, const double* row_sqnorm);

/* ---- A3: the fused dual-gradient pass ---------- */
#define DL_GRAD_PARTIAL 1u /* grad = A_shard x* (no -b); obj = {c^T x, reg, nnz(x), 0} partials */
/* lambda: device [m*J] float32 dual point (original coordinates, >= 0 expected);
 * gamma > 0; grad: device [m*J] fp64 = A x*(lambda) - b;
 * obj: device [4] fp64 = { g(lambda), c^T x*, (gamma/2) x*^T D_v^2 x*, nnz(x*) }. */
dl_status dl_dual_grad(dl_problem* p, const float* lambda, double gamma, double* grad, double* obj,
                       uint32_t flags);
/* Same with HOST buffers: lambda host [m*J], grad host [m*J], obj host [4]; copies
 * inside the call; synchronous. */
dl_status dl_dual_grad_host(dl_problem* p, const float* lambda, double gamma, double* grad, double* obj,
                            uint32_t flags);
/* x*(lambda) in the ORIGINAL edge order: x device [nnz] float32. */
dl_status dl_primal(dl_problem* p, const float* lambda, double gamma, float* x);

/* ---- A4: AGD with adaptive step and gamma continuation */
typedef struct {
  double gamma0;       /* initial ridge parameter (> 0)                                   */
  double gamma_min;    /* continuation floor; <= 0 or == gamma0 means fixed gamma          */
  int32_t halve_every; /* gamma halves every this many iterations (25)       */
  int32_t use_jacobi;  /* apply D from dl_set_jacobi                                        */
  double max_step;     /* max-step-size at gamma_ref (1e-3), R6    */
  double init_step;    /* initial-step-size (1e-5)                           */
  int64_t history_cap; /* iteration records kept on device (0: 65536)                       */
} dl_agd_params;

typedef struct {
  int64_t iter;   /* t                                   */
  double g;       /* g(mu_t), mu_t = fl32(D lam2_t)       */
  double gamma;   /* gamma_t                              */
  double eta;     /* step used at t                       */
  double gnorm;   /* ||D (A x - b)||                      */
  double infeas;  /* ||(A x - b)_+||  (Appendix A.2)       */
  double nnz_x;   /* nonzeros of x*(mu_t)                 */
} dl_iter_record;

/* Resets the state: lam1 = lam2 = 0, t = 0, gamma = gamma0. */
dl_status dl_agd_init(dl_problem* p, const dl_agd_params* prm);
/* Runs the fused pass at the state's point mu_t (every CTA into its own accumulator copy, then
 * the copies summed in CTA order, R16) and leaves the result in the problem's
 * accumulator, overwriting it (local shard only: all-reduce `acc` across ranks before
 * dl_dual_step). */
dl_status dl_agd_eval(dl_problem* p);
/* acc: device fp64 [m*J + 4] = {A x (m*J), c^T x, reg, nnz(x), 0}; count returned in n.
 * The m*J part is indexed by destination LABEL (k*J + lab[j]); all-reduce it as is. */
dl_status dl_agd_accumulator(dl_problem* p, double** acc, int64_t* n);
/* The solver's accumulated gradient at the current point mu_t, after dl_agd_eval (and, when
 * sharded, the all-reduce of the accumulator) and before dl_dual_step: grad [m*J] fp64 =
 * A x*(mu_t) - b in ORIGINAL order, obj [4] = {g(mu_t), c^T x*, reg, nnz(x*)}; device pointers. */
dl_status dl_agd_gradient(dl_problem* p, double* grad, double* obj);
/* One AGD step (R5-R8) from the accumulated gradient; resets the pass's work
 * counters and appends one history record, a dl_iter_record; the next dl_agd_eval overwrites
 * the accumulator. */
dl_status dl_dual_step(dl_problem* p);
/* `iters` iterations of eval -> [NCCL all-reduce if dl_comm_init] -> step, captured
 * in a CUDA graph.  Asynchronous; read results with dl_agd_history / dl_agd_dual. */
dl_status dl_solve(dl_problem* p, int64_t iters);
/* The dual point mu_t = fl32(D lam2_t) the next dl_agd_eval evaluates (ORIGINAL coordinates,
 * float32 [m*J], device or host auto-detected; host copies are synchronous). */
dl_status dl_agd_point(dl_problem* p, float* mu_out);
/* Copies records [0, min(cap, t)) to HOST; *count = records available. Synchronous. */
dl_status dl_agd_history(dl_problem* p, dl_iter_record* out, int64_t cap, int64_t* count);
/* Current duals, device or host (auto-detected), fp64 [m*J] in ORIGINAL coordinates:
 * lam1_out = D lam1 (the iterate), lam2_out = D lam2 (extrapolated point); NULL skips. */
dl_status dl_agd_dual(dl_problem* p, double* lam1_out, double* lam2_out);

/* ---- A5: multi-GPU ------------------------------------ */
/* NCCL is loaded at run time (dlopen "libnccl.so.2").  Rank 0 calls
 * dl_comm_unique_id (128 bytes, host), shares it (e.g. torch.distributed
 * broadcast), then every rank calls dl_comm_init.  dl_solve then all-reduces
 * the m*J+4 accumulator once per iteration.  world == 1 creates a real one-rank
 * communicator (the same code path; the all-reduce is then the identity).
 * dl_comm_init all-reduces the destination edge counts and relabels every rank's
 * layout with the GLOBAL labels (so the accumulators agree across ranks); it resets the
 * AGD state (call dl_agd_init afterwards).  Calling it again replaces the communicator. */
dl_status dl_comm_unique_id(void* id128);
dl_status dl_comm_init(dl_problem* p, int32_t rank, int32_t world, const void* id128);
/* In-place sum all-reduce of a device fp64 buffer over the problem's communicator
 * (used for row norms / greedy loads at setup). */
dl_status dl_comm_allreduce(dl_problem* p, double* buf, int64_t n);

/* Diagnostics: with DUALIP_TRACE=1 in the environment at create time, every fused pass records
 * per CTA {smid, globaltimer at start, after lambda staging, at exit (ns), tiles worked}
 * (5 x uint64 per CTA), then the globaltimer at which each 4-tile chunk of the short-block phase was
 * finished (written by the pass itself: the last pass only).  *n = the record count (0 when tracing
 * is off); copies min(cap, *n) to the HOST buffer out (NULL: size query only).  Synchronous. */
dl_status dl_debug_trace(dl_problem* p, uint64_t* out, int64_t cap, int64_t* n);

/* Measurement: record the caller's CUDA events (cudaEvent_t, created by the caller) on the problem's
 * stream immediately before (start) and after (stop) every fused-pass kernel launched outside graph
 * capture (dl_agd_eval, dl_dual_grad*, dl_primal), so that the pass alone can be timed with
 * cudaEventElapsedTime; the events are overwritten by each pass.  NULL, NULL stops recording.
 * Both or neither must be given (DL_ERR_INVALID otherwise). */
dl_status dl_set_pass_events(dl_problem* p, void* start, void* stop);

/* Synchronise the problem's stream. */
dl_status dl_sync(dl_problem* p);

#ifdef __cplusplus
}
#endif
#endif /* DUALIP_H */
