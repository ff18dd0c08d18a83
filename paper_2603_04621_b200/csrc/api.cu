// C ABI (include/dualip.h): problem lifetime, layout build, gradient / AGD / solve
// entry points, CUDA-graph capture of the iteration, NCCL (dlopen) all-reduce.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

// Minimal NCCL surface (types from nccl.h; functions resolved with dlsym).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclUint64 = 5, kNcclFloat64 = 8, kNcclSum = 0 };

namespace dl {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
static Nccl g_nccl;

static bool load_nccl() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error(std::string("NCCL not loadable (dlopen libnccl.so.2): ") + dlerror());
    return false;
  }
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy;
  if (!g_nccl.ok) set_error("NCCL symbols missing");
  return g_nccl.ok;
}

}  // namespace dl

using namespace dl;

struct dl_problem {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t I = 0, nnz = 0;
  int32_t J = 0, M = 1, kind = 0;
  double r = 1.0, u = INFINITY;
  // layout
  Plan plan;
  int32_t tile_cap = 256, lam_mode = kLamSmem, lam_hot = 0, num_sms = 148, ctas = 148;
  size_t smem = 0;
  int64_t nnz_layout = 0, a_stride = 0;
  int32_t* d_dest = nullptr;  // destination LABELS
  float *d_c = nullptr, *d_a = nullptr, *d_b = nullptr, *d_vsq = nullptr, *d_vinv = nullptr;  // d_b by label
  Tile* d_tiles = nullptr;
  uint16_t* d_blk_rel = nullptr;
  uint16_t* d_rel_pool = nullptr;
  int64_t* d_orig_off = nullptr;
  double* d_gscratch = nullptr;
  int64_t gscratch_per_cta = 0;
  unsigned long long* d_trace = nullptr;  // per-CTA launch trace of the last fused pass (DUALIP_TRACE=1)
  cudaEvent_t ev_pass[2] = {nullptr, nullptr};  // caller's events around every fused launch (dl_set_pass_events)
  // destination labels (R15): lab[j] = label of j, unlab = inverse
  bool relabeled = false;
  int32_t *d_lab = nullptr, *d_unlab = nullptr;
  std::vector<int32_t> lab;
  std::vector<unsigned long long> counts;  // this shard's edges per destination (relabeled problems)
  double* d_step_part = nullptr;  // AGD step: per-CTA partials, completion counter, eta/beta
  int32_t* d_step_done = nullptr;
  double* d_step_scal = nullptr;
  // solver work (AGD accumulator) and standalone-gradient work: separate buffers, so a
  // standalone call between solver steps never disturbs the solver's accumulator
  double* d_part = nullptr;  // per-CTA partial accumulators [part_copies][part_stride] (zero between passes)
  int64_t part_stride = 0;
  int32_t part_copies = 1;
  double* d_acc = nullptr;   // [MJ + 4]
  int32_t* d_ctr = nullptr;  // [8]
  double* d_acc_s = nullptr;
  int32_t* d_ctr_s = nullptr;
  // standalone grad path
  float* d_lam_in = nullptr;   // caller lambda (host entry), ORIGINAL order
  float* d_lam_lab = nullptr;  // lambda in label order
  double *d_grad_out = nullptr, *d_obj_out = nullptr;
  double* d_tmp = nullptr;     // [MJ] relabel scratch
  // Jacobi
  double* d_D = nullptr;       // by label
  double* d_Dones = nullptr;
  bool jacobi_set = false;
  // AGD
  bool agd_ready = false;
  dl_agd_params prm{};
  double *d_lam1 = nullptr, *d_lam2 = nullptr, *d_lam2_prev = nullptr, *d_G_prev = nullptr;
  float* d_mu = nullptr;
  AgdDev* d_st = nullptr;
  dl_iter_record* d_hist = nullptr;
  int64_t hist_cap = 0;
  // graph
  cudaGraphExec_t graph = nullptr;
  int graph_iters = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  int32_t rank = 0, world = 1;
  int64_t device_bytes = 0;
  std::vector<void*> allocs;
};

namespace {

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                         \
      return _e == cudaErrorMemoryAllocation ? DL_ERR_OOM : DL_ERR_CUDA;                      \
    }                                                                                        \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
dl_status dev_alloc(dl_problem* p, T** ptr, size_t count) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    cudaGetLastError();
    return DL_ERR_OOM;
  }
  p->allocs.push_back(q);
  p->device_bytes += (int64_t)bytes;
  *ptr = static_cast<T*>(q);
  return DL_OK;
}

#define DL_TRY(expr)                  \
  do {                                \
    dl_status _s = (expr);            \
    if (_s != DL_OK) return _s;       \
  } while (0)

void dev_release(dl_problem* p, void* q, size_t bytes) {
  if (!q) return;
  cudaFree(q);
  auto it = std::find(p->allocs.begin(), p->allocs.end(), q);
  if (it != p->allocs.end()) p->allocs.erase(it);
  p->device_bytes -= (int64_t)bytes;
}

void free_all(dl_problem* p) {
  if (p->graph) cudaGraphExecDestroy(p->graph);
  p->graph = nullptr;
  for (void* q : p->allocs) cudaFree(q);
  p->allocs.clear();
  if (p->comm && g_nccl.ok) g_nccl.CommDestroy(p->comm);
  p->comm = nullptr;
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
}

// Labels by edge count, descending, ties by destination index (R15).
std::vector<int32_t> labels_from_counts(const std::vector<unsigned long long>& cnt) {
  const int32_t J = (int32_t)cnt.size();
  std::vector<int32_t> order(J);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return cnt[x] > cnt[y]; });
  std::vector<int32_t> lab(J);
  for (int32_t l = 0; l < J; ++l) lab[order[l]] = l;
  return lab;
}

GradArgs grad_args(dl_problem* p, const float* lam, const double* gamma_ptr, double gamma_val, float* x_out,
                   int32_t* ctr) {
  GradArgs a{};
  a.dest = p->d_dest;
  a.c = p->d_c;
  a.a = p->d_a;
  a.a_stride = p->a_stride;
  a.tiles = p->d_tiles;
  for (int i = 0; i < kNumBigPhases + 2; ++i) a.ph_begin[i] = p->plan.ph_begin[i];
  a.blk_rel = p->d_blk_rel;
  a.rel_pool = p->d_rel_pool;
  a.vsq = p->d_vsq;
  a.vinv = p->d_vinv;
  a.orig_off = p->d_orig_off;
  a.lam = lam;
  a.J = p->J;
  a.m = p->M;
  a.gamma_ptr = gamma_ptr;
  a.gamma_val = gamma_val;
  a.r = p->r;
  a.u = p->u;
  a.kind = p->kind;
  a.tile_cap = p->tile_cap;
  a.lam_mode = p->lam_mode;
  a.lam_hot = p->lam_hot;
  a.acc = p->d_part;
  a.acc_stride = p->part_stride;
  a.acc_copies = p->part_copies;
  a.num_sms = p->num_sms;
  a.ctr = ctr;
  a.x_out = x_out;
  a.gscratch = p->d_gscratch;
  a.gscratch_per_cta = p->gscratch_per_cta;
  a.trace = p->d_trace;
  return a;
}

// Fused pass at lam (label order) into acc/ctr: the solver's buffers (never zeroed here: the
// step kernel resets them) or the standalone ones (zeroed first).
dl_status run_grad(dl_problem* p, const float* lam, const double* gamma_ptr, double gamma_val, float* x_out,
                   bool standalone) {
  const int64_t n = (int64_t)p->M * p->J;
  double* acc = standalone ? p->d_acc_s : p->d_acc;
  int32_t* ctr = standalone ? p->d_ctr_s : p->d_ctr;
  if (standalone) CUDA_TRY(cudaMemsetAsync(ctr, 0, 8 * sizeof(int32_t), p->stream));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool evs = p->ev_pass[0] && cudaStreamIsCapturing(p->stream, &cap) == cudaSuccess &&
                   cap == cudaStreamCaptureStatusNone;
  if (evs) CUDA_TRY(cudaEventRecord(p->ev_pass[0], p->stream));
  if (!p->plan.tiles.empty())
    CUDA_TRY(launch_fused_grad(grad_args(p, lam, gamma_ptr, gamma_val, x_out, ctr), p->ctas, p->smem,
                               p->stream));
  if (evs) CUDA_TRY(cudaEventRecord(p->ev_pass[1], p->stream));
  // the CTA copies -> acc (every row written; the copies are left zero for the next pass)
  CUDA_TRY(launch_partial_sum(p->d_part, p->part_stride, p->part_copies, n + 4, acc, p->stream));
  return DL_OK;
}

// lambda (ORIGINAL order, device) -> label order for the fused pass
const float* lam_to_labels(dl_problem* p, const float* lam, cudaError_t* err) {
  *err = cudaSuccess;
  if (!p->relabeled) return lam;
  *err = launch_permute_f32(lam, p->d_lab, p->d_lam_lab, p->M, p->J, 0, p->stream);
  return p->d_lam_lab;
}

StepArgs step_args(dl_problem* p) {
  StepArgs s{};
  s.n = p->M * p->J;
  s.D = p->prm.use_jacobi ? p->d_D : p->d_Dones;
  s.b = p->d_b;
  s.acc = p->d_acc;
  s.ctr = p->d_ctr;
  s.lam1 = p->d_lam1;
  s.lam2 = p->d_lam2;
  s.lam2_prev = p->d_lam2_prev;
  s.G_prev = p->d_G_prev;
  s.mu = p->d_mu;
  s.st = p->d_st;
  s.hist = p->d_hist;
  s.part = p->d_step_part;
  s.done = p->d_step_done;
  s.scal = p->d_step_scal;
  return s;
}

dl_status enqueue_iteration(dl_problem* p) {
  DL_TRY(run_grad(p, p->d_mu, &p->d_st->gamma, 0.0, nullptr, false));
  if (p->comm) {
    ncclResult_t r = g_nccl.AllReduce(p->d_acc, p->d_acc, (size_t)p->M * p->J + 4, kNcclFloat64, kNcclSum,
                                      p->comm, p->stream);
    if (r != 0) {
      set_error(std::string("ncclAllReduce: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
      return DL_ERR_NCCL;
    }
  }
  CUDA_TRY(launch_agd_step(step_args(p), p->stream));
  return DL_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int dl_abi_version(void) { return DL_ABI_VERSION; }
const char* dl_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace {

// Shared body of dl_problem_create (device input) and dl_problem_create_host (host input).
dl_status create_common(const dl_problem_desc* d, dl_problem** out, bool host) {
  const char* fn = host ? "dl_problem_create_host" : "dl_problem_create";
  if (!d || !out) {
    set_error(std::string(fn) + ": NULL argument");
    return DL_ERR_INVALID;
  }
  *out = nullptr;
  if (d->num_sources < 0 || d->num_dests < 1 || d->num_families < 1 || d->num_families > 4 || d->nnz < 0 ||
      (d->num_sources > 0 && !d->row_ptr) || (d->nnz > 0 && (!d->dest || !d->a || !d->c)) || !d->b ||
      d->nnz >= (1LL << 40) || d->num_sources >= (1LL << 31) || (int64_t)d->num_families * d->num_dests >= (1 << 30)) {
    set_error(std::string(fn) + ": invalid sizes or NULL arrays");
    return DL_ERR_INVALID;
  }
  if (d->proj_kind < DL_PROJ_SIMPLEX || d->proj_kind > DL_PROJ_BOX) {
    set_error(std::string(fn) + ": unknown proj_kind");
    return DL_ERR_INVALID;
  }
  if ((d->proj_kind != DL_PROJ_BOX && !(d->proj_r > 0)) || (d->proj_kind != DL_PROJ_SIMPLEX && !(d->proj_u > 0))) {
    set_error(std::string(fn) + ": caps must be positive (r for simplex/box-cut, u for box-cut/box)");
    return DL_ERR_INVALID;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || d->device < 0 || d->device >= ndev) {
    cudaGetLastError();
    set_error(std::string(fn) + ": no CUDA device (there is no CPU fallback)");
    return DL_ERR_CUDA;
  }
  DeviceGuard guard(d->device);
  dl_problem* p = new dl_problem();
  p->device = d->device;
  p->I = d->num_sources;
  p->nnz = d->nnz;
  p->J = d->num_dests;
  p->M = d->num_families;
  p->kind = d->proj_kind;
  p->r = d->proj_kind == DL_PROJ_BOX ? INFINITY : d->proj_r;
  p->u = d->proj_kind == DL_PROJ_SIMPLEX ? INFINITY : d->proj_u;
  auto fail = [&](dl_status s) {
    free_all(p);
    delete p;
    return s;
  };
#define CREATE_TRY(expr)                                                   \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      set_error(std::string(fn) + ": " #expr ": " + cudaGetErrorString(_e)); \
      cudaGetLastError();                                                  \
      return fail(_e == cudaErrorMemoryAllocation ? DL_ERR_OOM : DL_ERR_CUDA); \
    }                                                                      \
  } while (0)
  if (d->stream) {
    p->stream = (cudaStream_t)d->stream;
  } else {
    CREATE_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
  }
  cudaDeviceProp prop;
  CREATE_TRY(cudaGetDeviceProperties(&prop, p->device));
  p->num_sms = prop.multiProcessorCount;
  p->ctas = p->num_sms;
  const SmemRule rule = smem_rule(p->M, p->J, p->kind);
  p->tile_cap = rule.tile_cap;
  p->lam_mode = rule.lam_mode;
  p->lam_hot = rule.hot;
  p->relabeled = rule.lam_mode != kLamSmem;
  p->smem = fused_smem_bytes(p->M, p->kind, p->tile_cap, p->lam_mode == kLamGlobal ? 0 : p->lam_hot);
  if ((size_t)prop.sharedMemPerBlockOptin < p->smem) {
    set_error(std::string(fn) + ": device shared memory per block below the layout's need");
    return fail(DL_ERR_UNSUPPORTED);
  }
  // ---- row_ptr on the host, plan
  std::vector<int64_t> rp_copy;
  const int64_t* rp = nullptr;
  if (host) {
    rp = p->I > 0 ? d->row_ptr : nullptr;
  } else {
    rp_copy.assign((size_t)p->I + 1, 0);
    if (p->I > 0) {
      CREATE_TRY(cudaMemcpyAsync(rp_copy.data(), d->row_ptr, rp_copy.size() * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, p->stream));
      CREATE_TRY(cudaStreamSynchronize(p->stream));
    }
    rp = rp_copy.data();
  }
  static const int64_t kZero[1] = {0};
  if (!rp) rp = kZero;
  if (rp[0] != 0 || rp[(size_t)p->I] != p->nnz) {
    set_error(std::string(fn) + ": row_ptr[0] != 0 or row_ptr[I] != nnz");
    return fail(DL_ERR_INVALID);
  }
  for (int64_t i = 0; i < p->I; ++i)
    if (rp[i + 1] < rp[i]) {
      set_error(std::string(fn) + ": row_ptr decreasing");
      return fail(DL_ERR_INVALID);
    }
  p->plan = make_plan(rp, p->I, p->tile_cap);
  const Plan& P = p->plan;
  const int64_t nb = (int64_t)P.perm.size(), nt = (int64_t)P.tiles.size();
  p->nnz_layout = P.total;
  p->a_stride = (P.total + 2 * kAlign + 31) / 32 * 32;  // room for the last tile's rounded copy
  const int64_t MJ = (int64_t)p->M * p->J;
  const int64_t J = p->J;
  // ---- device buffers
  dl_status s;
  if ((s = dev_alloc(p, &p->d_dest, p->a_stride)) || (s = dev_alloc(p, &p->d_c, p->a_stride)) ||
      (s = dev_alloc(p, &p->d_a, (size_t)p->a_stride * p->M)) || (s = dev_alloc(p, &p->d_b, MJ)) ||
      (s = dev_alloc(p, &p->d_tiles, nt + 8)) || (s = dev_alloc(p, &p->d_blk_rel, nb)) ||
      (s = dev_alloc(p, &p->d_orig_off, nb)) || (s = dev_alloc(p, &p->d_acc, MJ + 4)) ||
      (s = dev_alloc(p, &p->d_ctr, 8)) || (s = dev_alloc(p, &p->d_acc_s, MJ + 4)) ||
      (s = dev_alloc(p, &p->d_ctr_s, 8)) || (s = dev_alloc(p, &p->d_D, MJ)) || (s = dev_alloc(p, &p->d_Dones, MJ)) ||
      (s = dev_alloc(p, &p->d_lam_in, MJ)) || (s = dev_alloc(p, &p->d_lam_lab, MJ)) ||
      (s = dev_alloc(p, &p->d_grad_out, MJ)) || (s = dev_alloc(p, &p->d_obj_out, 4)) ||
      (s = dev_alloc(p, &p->d_tmp, MJ)) || (s = dev_alloc(p, &p->d_lab, J)) || (s = dev_alloc(p, &p->d_unlab, J)))
    return fail(s);
  if (d->v && ((s = dev_alloc(p, &p->d_vsq, nb)) || (s = dev_alloc(p, &p->d_vinv, nb)))) return fail(s);
  // accumulator copies: one per CTA while all of them fit in
  // 16 MB of L2 (m J <= ~13.5k); fewer for larger m J, each shared by a run of neighbouring SMs
  // (more would not stay in L2: the reductions would then read-modify-write DRAM)
  p->part_stride = (MJ + 4 + 31) / 32 * 32;
  int64_t copies = std::max<int64_t>(1, std::min<int64_t>(p->ctas, (int64_t)(16ll << 20) / (p->part_stride * 8)));
  if (const char* e = std::getenv("DUALIP_ACC_COPIES")) {  // tuning experiments
    const int64_t v = std::atoll(e);
    if (v >= 1 && v <= p->ctas) copies = v;
  }
  p->part_copies = (int32_t)copies;
  if ((s = dev_alloc(p, &p->d_part, (size_t)p->part_stride * p->part_copies))) return fail(s);
  CREATE_TRY(cudaMemsetAsync(p->d_part, 0, (size_t)p->part_stride * p->part_copies * sizeof(double), p->stream));
  // global d-scratch for blocks longer than a 16-warp group's shared scratch
  const int64_t smem_scr = (int64_t)kWarps * 2 * p->tile_cap * (8 + 4 * p->M) / 8;  // fp64 d
  if (P.max_len > smem_scr) {
    p->gscratch_per_cta = P.max_len;
    if ((s = dev_alloc(p, &p->d_gscratch, (size_t)P.max_len * p->ctas))) return fail(s);
  }
  // ---- destination labels (R15): popularity order when lambda is not fully on chip
  p->lab.resize((size_t)J);
  if (p->relabeled) {
    p->counts.assign((size_t)J, 0ull);
    if (host) {
      const int nth = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
      std::vector<std::vector<unsigned long long>> part((size_t)nth, std::vector<unsigned long long>((size_t)J, 0));
      std::vector<int> badf((size_t)nth, 0);
      std::vector<std::thread> th;
      for (int t = 0; t < nth; ++t)
        th.emplace_back([&, t]() {
          const int64_t e0 = p->nnz * t / nth, e1 = p->nnz * (t + 1) / nth;
          auto& c = part[(size_t)t];
          for (int64_t e = e0; e < e1; ++e) {
            const uint32_t j = (uint32_t)d->dest[e];
            if (j < (uint32_t)J) c[j]++;
            else badf[(size_t)t] = 1;
          }
        });
      for (auto& x : th) x.join();
      for (int t = 0; t < nth; ++t) {
        if (badf[(size_t)t]) {
          set_error(std::string(fn) + ": a dest index is outside [0, num_dests)");
          return fail(DL_ERR_INVALID);
        }
        for (int64_t j = 0; j < J; ++j) p->counts[(size_t)j] += part[(size_t)t][(size_t)j];
      }
    } else {
      unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(p->d_tmp);  // MJ doubles >= J counts
      CREATE_TRY(cudaMemsetAsync(d_cnt, 0, (size_t)J * 8, p->stream));
      CREATE_TRY(launch_dest_histogram(d->dest, p->nnz, p->J, d_cnt, p->stream));
      CREATE_TRY(cudaMemcpyAsync(p->counts.data(), d_cnt, (size_t)J * 8, cudaMemcpyDeviceToHost, p->stream));
      CREATE_TRY(cudaStreamSynchronize(p->stream));
    }
    p->lab = labels_from_counts(p->counts);
  } else {
    std::iota(p->lab.begin(), p->lab.end(), 0);
  }
  {
    std::vector<int32_t> unlab((size_t)J);
    for (int64_t j = 0; j < J; ++j) unlab[(size_t)p->lab[(size_t)j]] = (int32_t)j;
    CREATE_TRY(cudaMemcpyAsync(p->d_lab, p->lab.data(), (size_t)J * 4, cudaMemcpyHostToDevice, p->stream));
    CREATE_TRY(cudaMemcpyAsync(p->d_unlab, unlab.data(), (size_t)J * 4, cudaMemcpyHostToDevice, p->stream));
    CREATE_TRY(cudaStreamSynchronize(p->stream));  // unlab is a stack vector
  }
  // ---- host -> device plan arrays
  std::vector<uint16_t> rel((size_t)nb, 0);
  std::vector<int64_t> orig((size_t)nb, 0);
  std::vector<uint16_t> pool;
  for (Tile& tl : p->plan.tiles) {
    for (int q = 0; q < tl.nb; ++q) rel[tl.b0 + q] = (uint16_t)(tl.bucket >= kBigBucket ? 0 : P.blk_off[tl.b0 + q] - tl.off);
    if (tl.bucket < kBigBucket && tl.nb < kRelMax) {  // 16-B slot {rel_0..rel_{nb-1}, nnz} streamed with the tile
      tl.rel_off = (int32_t)pool.size();
      for (int q = 0; q < tl.nb; ++q) pool.push_back(rel[tl.b0 + q]);
      pool.push_back((uint16_t)tl.nnz);
      while (pool.size() % 8) pool.push_back(0);
    }
  }
  pool.resize(pool.size() + 64, 0);
  std::vector<int32_t> blk_of_src((size_t)p->I, -1);
  for (int64_t b = 0; b < nb; ++b) {
    orig[b] = rp[P.perm[b]];
    blk_of_src[(size_t)P.perm[b]] = (int32_t)b;
  }
  CREATE_TRY(cudaMemsetAsync(p->d_dest, 0, p->a_stride * sizeof(int32_t), p->stream));
  CREATE_TRY(cudaMemsetAsync(p->d_c, 0, p->a_stride * sizeof(float), p->stream));
  CREATE_TRY(cudaMemsetAsync(p->d_a, 0, (size_t)p->a_stride * p->M * sizeof(float), p->stream));
  if ((s = dev_alloc(p, &p->d_rel_pool, pool.size()))) return fail(s);
  CREATE_TRY(cudaMemsetAsync(p->d_tiles, 0, (nt + 8) * sizeof(Tile), p->stream));
  CREATE_TRY(cudaMemcpyAsync(p->d_tiles, P.tiles.data(), nt * sizeof(Tile), cudaMemcpyHostToDevice, p->stream));
  CREATE_TRY(cudaMemcpyAsync(p->d_rel_pool, pool.data(), pool.size() * sizeof(uint16_t), cudaMemcpyHostToDevice,
                             p->stream));
  CREATE_TRY(cudaMemcpyAsync(p->d_blk_rel, rel.data(), nb * sizeof(uint16_t), cudaMemcpyHostToDevice, p->stream));
  CREATE_TRY(cudaMemcpyAsync(p->d_orig_off, orig.data(), nb * sizeof(int64_t), cudaMemcpyHostToDevice, p->stream));
  // temporaries of the scatter: block of each source, block offsets, (host input) row_ptr + staging
  int32_t* d_bos = nullptr;
  int64_t *d_boff = nullptr, *d_rp = nullptr;
  int32_t* d_bad = nullptr;
  std::vector<std::pair<void*, size_t>> temps;
  auto tmp_alloc = [&](auto** ptr, size_t count) {
    dl_status st = dev_alloc(p, ptr, count);
    if (st == DL_OK) temps.push_back({(void*)*ptr, std::max<size_t>(count, 1) * sizeof(**ptr)});
    return st;
  };
  if ((s = tmp_alloc(&d_bos, (size_t)p->I)) || (s = tmp_alloc(&d_boff, (size_t)nb)) || (s = tmp_alloc(&d_bad, 1)))
    return fail(s);
  CREATE_TRY(cudaMemcpyAsync(d_bos, blk_of_src.data(), (size_t)p->I * 4, cudaMemcpyHostToDevice, p->stream));
  CREATE_TRY(cudaMemcpyAsync(d_boff, P.blk_off.data(), nb * sizeof(int64_t), cudaMemcpyHostToDevice, p->stream));
  CREATE_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), p->stream));
  LayoutArgs la{};
  la.a_stride_out = p->a_stride;
  la.m = p->M;
  la.blk_of_src = d_bos;
  la.blk_off = d_boff;
  la.lab = p->d_lab;
  la.dest_out = p->d_dest;
  la.c_out = p->d_c;
  la.a_out = p->d_a;
  la.vsq_out = p->d_vsq;
  la.vinv_out = p->d_vinv;
  la.J = p->J;
  la.bad = d_bad;
  if (!host) {
    la.row_ptr = d->row_ptr;
    la.dest = d->dest;
    la.a = d->a;
    la.c = d->c;
    la.v = d->v;
    la.i0 = 0;
    la.i1 = p->I;
    la.e0 = 0;
    la.a_in_stride = p->nnz;
    CREATE_TRY(launch_build_layout(la, p->stream));
  } else if (p->I > 0) {
    // stream source chunks (<= kChunk entries and sources) through one device staging buffer
    constexpr int64_t kChunk = 1ll << 26;
    const int64_t ch = std::min<int64_t>(kChunk, std::max<int64_t>(p->nnz, 1));
    const int64_t chs = std::min<int64_t>(kChunk, p->I);
    int32_t* st_dest = nullptr;
    float *st_c = nullptr, *st_a = nullptr, *st_v = nullptr;
    if ((s = tmp_alloc(&d_rp, (size_t)p->I + 1)) || (s = tmp_alloc(&st_dest, (size_t)ch)) ||
        (s = tmp_alloc(&st_c, (size_t)ch)) || (s = tmp_alloc(&st_a, (size_t)ch * p->M)) ||
        (d->v && (s = tmp_alloc(&st_v, (size_t)chs))))
      return fail(s);
    CREATE_TRY(cudaMemcpyAsync(d_rp, rp, ((size_t)p->I + 1) * 8, cudaMemcpyHostToDevice, p->stream));
    la.row_ptr = d_rp;
    la.dest = st_dest;
    la.c = st_c;
    la.a = st_a;
    la.v = st_v;
    la.a_in_stride = ch;
    int64_t i0 = 0;
    while (i0 < p->I) {
      int64_t i1 = std::min<int64_t>(p->I, i0 + chs);
      if (rp[i1] - rp[i0] > ch) i1 = std::upper_bound(rp + i0, rp + i1 + 1, rp[i0] + ch) - rp - 1;
      i1 = std::max<int64_t>(i1, i0 + 1);  // a source longer than a chunk cannot occur (kChunk >> 2^31/...)
      const int64_t e0 = rp[i0], n = rp[i1] - rp[i0];
      // pageable sources: each copy waits for the previous scatter on the stream (staging reuse)
      if (n > 0) {
        CREATE_TRY(cudaMemcpyAsync(st_dest, d->dest + e0, n * 4, cudaMemcpyHostToDevice, p->stream));
        CREATE_TRY(cudaMemcpyAsync(st_c, d->c + e0, n * 4, cudaMemcpyHostToDevice, p->stream));
        for (int f = 0; f < p->M; ++f)
          CREATE_TRY(cudaMemcpyAsync(st_a + (size_t)f * ch, d->a + (size_t)f * p->nnz + e0, n * 4,
                                     cudaMemcpyHostToDevice, p->stream));
      }
      if (d->v) CREATE_TRY(cudaMemcpyAsync(st_v, d->v + i0, (i1 - i0) * 4, cudaMemcpyHostToDevice, p->stream));
      la.i0 = i0;
      la.i1 = i1;
      la.e0 = e0;
      CREATE_TRY(launch_build_layout(la, p->stream));
      CREATE_TRY(cudaStreamSynchronize(p->stream));
      i0 = i1;
    }
  }
  {
    int32_t bad = 0;
    CREATE_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, p->stream));
    CREATE_TRY(cudaStreamSynchronize(p->stream));
    if (bad) {
      set_error(std::string(fn) + ": a dest index is outside [0, num_dests)");
      return fail(DL_ERR_INVALID);
    }
  }
  // b into label order
  {
    float* b_in = reinterpret_cast<float*>(p->d_tmp);
    CREATE_TRY(cudaMemcpyAsync(b_in, d->b, MJ * sizeof(float), host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                               p->stream));
    CREATE_TRY(launch_permute_f32(b_in, p->d_lab, p->d_b, p->M, p->J, 0, p->stream));
  }
  CREATE_TRY(launch_jacobi_diag(nullptr, p->d_lab, p->d_D, p->M, p->J, p->stream));
  CREATE_TRY(launch_jacobi_diag(nullptr, p->d_lab, p->d_Dones, p->M, p->J, p->stream));
  CREATE_TRY(cudaStreamSynchronize(p->stream));
  for (auto& t : temps) dev_release(p, t.first, t.second);
  if (const char* tr = std::getenv("DUALIP_TRACE"))
    if (tr[0] == '1' && (s = dev_alloc(p, &p->d_trace, (size_t)p->ctas * 5 + (size_t)nt / 4 + 8))) return fail(s);
#undef CREATE_TRY
  *out = p;
  return DL_OK;
}

// Relabel a problem with new labels (multi-rank: the global popularity order).  Remaps the
// layout's destinations and every label-ordered vector; the AGD state is reset.
dl_status relabel(dl_problem* p, const std::vector<int32_t>& lab_new) {
  if (lab_new == p->lab) return DL_OK;
  const int32_t J = p->J;
  std::vector<int32_t> unlab_new((size_t)J);
  for (int32_t j = 0; j < J; ++j) unlab_new[(size_t)lab_new[(size_t)j]] = j;
  int32_t *d_lab_new = nullptr, *d_unlab_new = nullptr;
  dl_status s;
  if ((s = dev_alloc(p, &d_lab_new, J)) || (s = dev_alloc(p, &d_unlab_new, J))) return s;
  CUDA_TRY(cudaMemcpyAsync(d_lab_new, lab_new.data(), (size_t)J * 4, cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY(cudaMemcpyAsync(d_unlab_new, unlab_new.data(), (size_t)J * 4, cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY(launch_relabel_dest(p->d_dest, p->nnz_layout, p->d_unlab, d_lab_new, p->stream));
  CUDA_TRY(launch_relabel_vec_f32(p->d_b, reinterpret_cast<float*>(p->d_tmp), p->d_unlab, d_lab_new, p->M, J,
                                  p->stream));
  CUDA_TRY(launch_relabel_vec_f64(p->d_D, p->d_tmp, p->d_unlab, d_lab_new, p->M, J, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  dev_release(p, p->d_lab, (size_t)J * 4);
  dev_release(p, p->d_unlab, (size_t)J * 4);
  p->d_lab = d_lab_new;
  p->d_unlab = d_unlab_new;
  p->lab = lab_new;
  p->agd_ready = false;
  if (p->graph) {
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
  }
  return DL_OK;
}

}  // namespace

extern "C" {

dl_status dl_problem_create(const dl_problem_desc* d, dl_problem** out) { return create_common(d, out, false); }
dl_status dl_problem_create_host(const dl_problem_desc* d, dl_problem** out) { return create_common(d, out, true); }

dl_status dl_problem_dest_labels(const dl_problem* p, int32_t* lab) {
  if (!p || !lab) {
    set_error("dl_problem_dest_labels: NULL argument");
    return DL_ERR_INVALID;
  }
  std::memcpy(lab, p->lab.data(), p->lab.size() * sizeof(int32_t));
  return DL_OK;
}

dl_status dl_problem_destroy(dl_problem* p) {
  if (!p) return DL_OK;
  DeviceGuard guard(p->device);
  cudaStreamSynchronize(p->stream);
  free_all(p);
  delete p;
  return DL_OK;
}

dl_status dl_problem_get_info(const dl_problem* p, dl_problem_info* o) {
  if (!p || !o) {
    set_error("dl_problem_get_info: NULL argument");
    return DL_ERR_INVALID;
  }
  std::memset(o, 0, sizeof(*o));
  o->num_sources = p->I;
  o->nnz = p->nnz;
  o->nnz_layout = p->nnz_layout;
  o->num_blocks = (int64_t)p->plan.perm.size();
  o->num_tiles = (int64_t)p->plan.tiles.size();
  o->num_big_tiles = p->plan.ph_begin[kNumBigPhases];
  o->num_dests = p->J;
  o->num_families = p->M;
  o->tile_cap = p->tile_cap;
  o->lambda_in_smem = p->lam_mode == kLamSmem;
  o->max_block_len = p->plan.max_len;
  o->num_buckets = p->plan.num_buckets;
  o->num_sms = p->num_sms;
  o->ctas = p->ctas;
  o->device_bytes = p->device_bytes;
  o->has_comm = p->comm != nullptr;
  o->comm_rank = p->rank;
  o->comm_world = p->world;
  o->relabeled = p->relabeled;
  o->lambda_hot = p->lam_mode == kLamGlobal ? 0 : p->lam_hot;
  return DL_OK;
}

dl_status dl_problem_layout(const dl_problem* p, int64_t* perm, int64_t* blk_off, int64_t* tiles) {
  if (!p) {
    set_error("dl_problem_layout: NULL problem");
    return DL_ERR_INVALID;
  }
  const Plan& P = p->plan;
  if (perm) std::memcpy(perm, P.perm.data(), P.perm.size() * sizeof(int64_t));
  if (blk_off) std::memcpy(blk_off, P.blk_off.data(), P.blk_off.size() * sizeof(int64_t));
  if (tiles) {
    // read the descriptors back from the device: the layout actually used
    std::vector<Tile> t(P.tiles.size());
    DeviceGuard guard(p->device);
    CUDA_TRY(cudaMemcpy(t.data(), p->d_tiles, t.size() * sizeof(Tile), cudaMemcpyDeviceToHost));
    for (size_t q = 0; q < t.size(); ++q) {
      tiles[5 * q + 0] = t[q].b0;
      tiles[5 * q + 1] = t[q].nb;
      tiles[5 * q + 2] = t[q].off;
      tiles[5 * q + 3] = t[q].nnz;
      tiles[5 * q + 4] = t[q].bucket;
    }
  }
  return DL_OK;
}

dl_status dl_problem_layout_data(const dl_problem* p, int32_t* dest, float* c, float* a) {
  if (!p) {
    set_error("dl_problem_layout_data: NULL problem");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  const size_t n = (size_t)p->nnz_layout;
  if (dest) {  // stored as labels: back to destination indices (gap entries hold label 0)
    CUDA_TRY(cudaMemcpy(dest, p->d_dest, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    std::vector<int32_t> unlab(p->lab.size());
    for (size_t j = 0; j < p->lab.size(); ++j) unlab[(size_t)p->lab[j]] = (int32_t)j;
    for (size_t e = 0; e < n; ++e) dest[e] = unlab[(size_t)dest[e]];
  }
  if (c) CUDA_TRY(cudaMemcpy(c, p->d_c, n * sizeof(float), cudaMemcpyDeviceToHost));
  if (a)
    for (int f = 0; f < p->M; ++f)
      CUDA_TRY(cudaMemcpy(a + f * n, p->d_a + f * p->a_stride, n * sizeof(float), cudaMemcpyDeviceToHost));
  return DL_OK;
}

dl_status dl_row_sqnorms(dl_problem* p, double* out) {
  if (!p || !out) {
    set_error("dl_row_sqnorms: NULL argument");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)p->M * p->J * sizeof(double), p->stream));
  CUDA_TRY(launch_row_sqnorms(p->d_dest, p->d_a, p->a_stride, p->nnz_layout, p->M, p->J, p->d_unlab, out, p->stream));
  return DL_OK;
}

dl_status dl_set_jacobi(dl_problem* p, const double* rowsq) {
  if (!p) {
    set_error("dl_set_jacobi: NULL problem");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  CUDA_TRY(launch_jacobi_diag(rowsq, p->d_lab, p->d_D, p->M, p->J, p->stream));
  p->jacobi_set = rowsq != nullptr;
  return DL_OK;
}

dl_status dl_dual_grad(dl_problem* p, const float* lam, double gamma, double* grad, double* obj, uint32_t flags) {
  if (!p || !lam || !grad || !obj || !(gamma > 0)) {
    set_error("dl_dual_grad: NULL argument or gamma <= 0");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  cudaError_t e;
  const float* lam_l = lam_to_labels(p, lam, &e);
  CUDA_TRY(e);
  DL_TRY(run_grad(p, lam_l, nullptr, gamma, nullptr, true));
  FinalizeArgs f{p->M * p->J, p->J, p->d_acc_s, p->d_b, lam_l, p->d_lab, grad, obj, (int32_t)(flags & DL_GRAD_PARTIAL)};
  CUDA_TRY(launch_finalize(f, p->stream));
  return DL_OK;
}

dl_status dl_dual_grad_host(dl_problem* p, const float* lam, double gamma, double* grad, double* obj,
                            uint32_t flags) {
  if (!p || !lam || !grad || !obj || !(gamma > 0)) {
    set_error("dl_dual_grad_host: NULL argument or gamma <= 0");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  const size_t n = (size_t)p->M * p->J;
  CUDA_TRY(cudaMemcpyAsync(p->d_lam_in, lam, n * sizeof(float), cudaMemcpyHostToDevice, p->stream));
  DL_TRY(dl_dual_grad(p, p->d_lam_in, gamma, p->d_grad_out, p->d_obj_out, flags));
  CUDA_TRY(cudaMemcpyAsync(grad, p->d_grad_out, n * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaMemcpyAsync(obj, p->d_obj_out, 4 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return DL_OK;
}

dl_status dl_primal(dl_problem* p, const float* lam, double gamma, float* x) {
  if (!p || !lam || !x || !(gamma > 0)) {
    set_error("dl_primal: NULL argument or gamma <= 0");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaMemsetAsync(x, 0, (size_t)p->nnz * sizeof(float), p->stream));
  cudaError_t e;
  const float* lam_l = lam_to_labels(p, lam, &e);
  CUDA_TRY(e);
  DL_TRY(run_grad(p, lam_l, nullptr, gamma, x, true));
  return DL_OK;
}

dl_status dl_agd_init(dl_problem* p, const dl_agd_params* prm) {
  if (!p || !prm || !(prm->gamma0 > 0) || !(prm->max_step > 0) || !(prm->init_step > 0) ||
      (prm->gamma_min > 0 && prm->gamma_min < prm->gamma0 && prm->halve_every < 1)) {
    set_error("dl_agd_init: invalid parameters");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  const int64_t n = (int64_t)p->M * p->J;
  if (!p->d_lam1) {  // allocate all or nothing (a failed attempt leaves no half-built state)
    double *l1 = nullptr, *l2 = nullptr, *l2p = nullptr, *gp = nullptr, *part = nullptr, *scal = nullptr;
    float* mu = nullptr;
    AgdDev* st = nullptr;
    int32_t* done = nullptr;
    const size_t before = p->allocs.size();
    dl_status s;
    if ((s = dev_alloc(p, &l1, n)) || (s = dev_alloc(p, &l2, n)) || (s = dev_alloc(p, &l2p, n)) ||
        (s = dev_alloc(p, &gp, n)) || (s = dev_alloc(p, &mu, n)) || (s = dev_alloc(p, &st, 1)) ||
        (s = dev_alloc(p, &part, 5 * kStepCtas)) || (s = dev_alloc(p, &done, 1)) || (s = dev_alloc(p, &scal, 2))) {
      while (p->allocs.size() > before) {
        cudaFree(p->allocs.back());
        p->allocs.pop_back();
      }
      return s;
    }
    CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(int32_t), p->stream));
    p->d_lam1 = l1;
    p->d_lam2 = l2;
    p->d_lam2_prev = l2p;
    p->d_G_prev = gp;
    p->d_mu = mu;
    p->d_st = st;
    p->d_step_part = part;
    p->d_step_done = done;
    p->d_step_scal = scal;
  }
  // the captured solve graph bakes in the history buffer and the Jacobi diagonal: rebuild it
  if (p->graph) {
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
  }
  const int64_t cap = prm->history_cap > 0 ? prm->history_cap : 65536;
  if (cap != p->hist_cap) {
    if (p->d_hist) {
      CUDA_TRY(cudaStreamSynchronize(p->stream));
      cudaFree(p->d_hist);
      p->allocs.erase(std::find(p->allocs.begin(), p->allocs.end(), (void*)p->d_hist));
      p->device_bytes -= std::max<int64_t>(p->hist_cap, 1) * (int64_t)sizeof(dl_iter_record);
      p->d_hist = nullptr;
    }
    dl_status s = dev_alloc(p, &p->d_hist, cap);
    if (s) return s;
    p->hist_cap = cap;
  }
  p->prm = *prm;
  AgdDev st{};
  const bool cont = prm->gamma_min > 0 && prm->gamma_min < prm->gamma0;
  st.gamma = prm->gamma0;
  st.gamma_prev = prm->gamma0;
  st.eta = prm->init_step;
  st.t = 0;
  st.k = 1;
  st.gamma0 = prm->gamma0;
  st.gamma_min = cont ? prm->gamma_min : prm->gamma0;
  st.gamma_ref = cont ? prm->gamma_min : prm->gamma0;
  st.max_step = prm->max_step;
  st.init_step = prm->init_step;
  st.halve_every = std::max(prm->halve_every, 1);
  st.continuation = cont ? 1 : 0;
  st.hist_cap = cap;
  CUDA_TRY(cudaMemcpyAsync(p->d_st, &st, sizeof(st), cudaMemcpyHostToDevice, p->stream));
  for (double* q : {p->d_lam1, p->d_lam2, p->d_lam2_prev, p->d_G_prev})
    CUDA_TRY(cudaMemsetAsync(q, 0, n * sizeof(double), p->stream));
  CUDA_TRY(cudaMemsetAsync(p->d_mu, 0, n * sizeof(float), p->stream));
  CUDA_TRY(cudaMemsetAsync(p->d_acc, 0, (n + 4) * sizeof(double), p->stream));
  CUDA_TRY(cudaMemsetAsync(p->d_ctr, 0, 8 * sizeof(int32_t), p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));  // st is a stack object
  p->agd_ready = true;
  return DL_OK;
}

dl_status dl_agd_eval(dl_problem* p) {
  if (!p || !p->agd_ready) {
    set_error("dl_agd_eval: call dl_agd_init first");
    return DL_ERR_STATE;
  }
  DeviceGuard guard(p->device);
  return run_grad(p, p->d_mu, &p->d_st->gamma, 0.0, nullptr, false);
}

dl_status dl_agd_accumulator(dl_problem* p, double** acc, int64_t* n) {
  if (!p || !acc || !n) {
    set_error("dl_agd_accumulator: NULL argument");
    return DL_ERR_INVALID;
  }
  *acc = p->d_acc;
  *n = (int64_t)p->M * p->J + 4;
  return DL_OK;
}

dl_status dl_agd_gradient(dl_problem* p, double* grad, double* obj) {
  if (!p || !p->agd_ready || !grad || !obj) {
    set_error("dl_agd_gradient: call dl_agd_init first / NULL output");
    return DL_ERR_STATE;
  }
  DeviceGuard guard(p->device);
  FinalizeArgs f{p->M * p->J, p->J, p->d_acc, p->d_b, p->d_mu, p->d_lab, grad, obj, 0};
  CUDA_TRY(launch_finalize(f, p->stream));
  return DL_OK;
}

dl_status dl_dual_step(dl_problem* p) {
  if (!p || !p->agd_ready) {
    set_error("dl_dual_step: call dl_agd_init first");
    return DL_ERR_STATE;
  }
  DeviceGuard guard(p->device);
  CUDA_TRY(launch_agd_step(step_args(p), p->stream));
  return DL_OK;
}

dl_status dl_solve(dl_problem* p, int64_t iters) {
  if (!p || !p->agd_ready) {
    set_error("dl_solve: call dl_agd_init first");
    return DL_ERR_STATE;
  }
  if (iters <= 0) return DL_OK;
  DeviceGuard guard(p->device);
  constexpr int kUnroll = 8;
  if (!p->graph) {
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
    dl_status s = DL_OK;
    for (int i = 0; i < kUnroll && s == DL_OK; ++i) s = enqueue_iteration(p);
    cudaError_t e = cudaStreamEndCapture(p->stream, &g);
    if (s != DL_OK) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    CUDA_TRY(e);
    e = cudaGraphInstantiate(&p->graph, g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(e);
    p->graph_iters = kUnroll;
  }
  int64_t full = iters / p->graph_iters, rem = iters % p->graph_iters;
  for (int64_t i = 0; i < full; ++i) CUDA_TRY(cudaGraphLaunch(p->graph, p->stream));
  for (int64_t i = 0; i < rem; ++i) DL_TRY(enqueue_iteration(p));
  return DL_OK;
}

dl_status dl_agd_history(dl_problem* p, dl_iter_record* outr, int64_t cap, int64_t* count) {
  if (!p || !p->agd_ready || !count) {
    set_error("dl_agd_history: not initialised or NULL count");
    return DL_ERR_STATE;
  }
  DeviceGuard guard(p->device);
  AgdDev st;
  CUDA_TRY(cudaMemcpyAsync(&st, p->d_st, sizeof(st), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  const int64_t avail = std::min(st.t, p->hist_cap);
  *count = st.t;
  if (outr && cap > 0) {
    const int64_t n = std::min(avail, cap);
    if (n > 0) CUDA_TRY(cudaMemcpy(outr, p->d_hist, n * sizeof(dl_iter_record), cudaMemcpyDeviceToHost));
  }
  return DL_OK;
}

dl_status dl_agd_dual(dl_problem* p, double* lam1_out, double* lam2_out) {
  if (!p || !p->agd_ready) {
    set_error("dl_agd_dual: call dl_agd_init first");
    return DL_ERR_STATE;
  }
  DeviceGuard guard(p->device);
  const double* D = p->prm.use_jacobi ? p->d_D : p->d_Dones;
  const int32_t n = p->M * p->J;
  double* outs[2] = {lam1_out, lam2_out};
  const double* src[2] = {p->d_lam1, p->d_lam2};
  for (int q = 0; q < 2; ++q) {
    if (!outs[q]) continue;
    cudaPointerAttributes at{};
    bool dev = cudaPointerGetAttributes(&at, outs[q]) == cudaSuccess && at.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    if (dev) {
      CUDA_TRY(launch_scale_out(D, src[q], p->d_lab, outs[q], p->M, p->J, p->stream));
    } else {
      CUDA_TRY(launch_scale_out(D, src[q], p->d_lab, p->d_grad_out, p->M, p->J, p->stream));
      CUDA_TRY(cudaMemcpyAsync(outs[q], p->d_grad_out, n * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
      CUDA_TRY(cudaStreamSynchronize(p->stream));
    }
  }
  return DL_OK;
}

dl_status dl_agd_point(dl_problem* p, float* mu_out) {
  if (!p || !p->agd_ready || !mu_out) {
    set_error("dl_agd_point: call dl_agd_init first / NULL output");
    return DL_ERR_STATE;
  }
  DeviceGuard guard(p->device);
  cudaPointerAttributes at{};
  const bool dev = cudaPointerGetAttributes(&at, mu_out) == cudaSuccess && at.type == cudaMemoryTypeDevice;
  cudaGetLastError();
  float* dst = dev ? mu_out : p->d_lam_in;
  CUDA_TRY(launch_permute_f32(p->d_mu, p->d_lab, dst, p->M, p->J, 1, p->stream));
  if (!dev) {
    CUDA_TRY(cudaMemcpyAsync(mu_out, dst, (size_t)p->M * p->J * sizeof(float), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
  }
  return DL_OK;
}

dl_status dl_comm_unique_id(void* id) {
  if (!id) {
    set_error("dl_comm_unique_id: NULL");
    return DL_ERR_INVALID;
  }
  if (!load_nccl()) return DL_ERR_NCCL;
  ncclUniqueId u;
  if (g_nccl.GetUniqueId(&u) != 0) {
    set_error("ncclGetUniqueId failed");
    return DL_ERR_NCCL;
  }
  std::memcpy(id, &u, sizeof(u));
  return DL_OK;
}

dl_status dl_comm_init(dl_problem* p, int32_t rank, int32_t world, const void* id) {
  if (!p || !id || world < 1 || rank < 0 || rank >= world) {
    set_error("dl_comm_init: bad arguments");
    return DL_ERR_INVALID;
  }
  if (!load_nccl()) return DL_ERR_NCCL;
  DeviceGuard guard(p->device);
  // a previous communicator / captured graph is replaced: drain the stream first
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  if (p->graph) {
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
  }
  if (p->comm) {
    g_nccl.CommDestroy(p->comm);
    p->comm = nullptr;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  ncclResult_t r = g_nccl.CommInitRank(&c, world, u, rank);  // world == 1: a real one-rank communicator
  if (r != 0) {
    set_error(std::string("ncclCommInitRank: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    return DL_ERR_NCCL;
  }
  p->comm = c;
  p->rank = rank;
  p->world = world;
  p->agd_ready = false;  // the accumulator layout may change below; dl_agd_init restarts the solver
  if (p->relabeled) {  // global popularity labels: all-reduce the per-destination edge counts
    unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(p->d_tmp);
    CUDA_TRY(cudaMemcpyAsync(d_cnt, p->counts.data(), (size_t)p->J * 8, cudaMemcpyHostToDevice, p->stream));
    r = g_nccl.AllReduce(d_cnt, d_cnt, (size_t)p->J, kNcclUint64, kNcclSum, p->comm, p->stream);
    if (r != 0) {
      set_error("ncclAllReduce (destination counts) failed");
      return DL_ERR_NCCL;
    }
    std::vector<unsigned long long> global((size_t)p->J);
    CUDA_TRY(cudaMemcpyAsync(global.data(), d_cnt, (size_t)p->J * 8, cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    DL_TRY(relabel(p, labels_from_counts(global)));
  }
  return DL_OK;
}

dl_status dl_comm_allreduce(dl_problem* p, double* buf, int64_t n) {
  if (!p || !buf || n < 0) {
    set_error("dl_comm_allreduce: bad arguments");
    return DL_ERR_INVALID;
  }
  if (!p->comm || n == 0) return DL_OK;
  DeviceGuard guard(p->device);
  ncclResult_t r = g_nccl.AllReduce(buf, buf, (size_t)n, kNcclFloat64, kNcclSum, p->comm, p->stream);
  if (r != 0) {
    set_error("ncclAllReduce failed");
    return DL_ERR_NCCL;
  }
  return DL_OK;
}

dl_status dl_debug_trace(dl_problem* p, uint64_t* out, int64_t cap, int64_t* n) {
  if (!p || !n) {
    set_error("dl_debug_trace: NULL");
    return DL_ERR_INVALID;
  }
  *n = p->d_trace ? (int64_t)p->ctas * 5 + (int64_t)p->plan.tiles.size() / 4 + 8 : 0;
  if (!p->d_trace || !out) return DL_OK;
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaMemcpyAsync(out, p->d_trace, (size_t)std::min(cap, *n) * 8, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return DL_OK;
}

dl_status dl_set_pass_events(dl_problem* p, void* start, void* stop) {
  if (!p || (!start) != (!stop)) {
    set_error("dl_set_pass_events: NULL problem, or only one event given");
    return DL_ERR_INVALID;
  }
  p->ev_pass[0] = (cudaEvent_t)start;
  p->ev_pass[1] = (cudaEvent_t)stop;
  return DL_OK;
}

dl_status dl_sync(dl_problem* p) {
  if (!p) {
    set_error("dl_sync: NULL");
    return DL_ERR_INVALID;
  }
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return DL_OK;
}

}  // extern "C"
