// Small kernels around the fused pass: AGD step (K2), gradient finalize (K3),
// Jacobi row norms (K4), layout build (K5).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "internal.h"

namespace dl {
namespace {

constexpr int kStepThreads = 1024;
constexpr int kRedThreads = 256;

// Deterministic block reduction of NV doubles (fixed tree over a fixed thread map).
template <int NV>
__device__ void block_sum(double (&v)[NV], double (*sm)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sm[i][warp] = v[i];
  __syncthreads();
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sm[i][w];
    v[i] = t;
  }
  __syncthreads();
}

__device__ __forceinline__ double gamma_at(const AgdDev& st, int64_t t) {
  if (!st.continuation) return st.gamma0;
  int64_t h = t / st.halve_every;
  double g = h > 2000 ? 0.0 : ldexp(st.gamma0, -(int)h);
  return fmax(g, st.gamma_min);
}

// One AGD iteration (R5-R8; oracle/agd.py steps 2-5) from the accumulated
// A x*(mu_t) (+ objective scalars), as two grid-wide kernels:
//  agd_reduce_kernel: CTA c reduces rows [c chunk, (c+1) chunk) to 5 partial sums (fixed
//   tree); the last CTA to finish adds the partials in CTA order, so the result does not
//   depend on scheduling and every rank computes identical bits; it then sets eta, beta,
//   the next gamma and the history record.
//  agd_update_kernel: lambda update (eta, beta from the reduce) and accumulator reset.
__global__ void __launch_bounds__(kRedThreads) agd_reduce_kernel(const StepArgs a) {
  __shared__ double sm[5][32];
  __shared__ bool last;
  const int n = a.n;
  const AgdDev st = *a.st;
  const int64_t t = st.t;
  const int chunk = (n + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  double v[5] = {0, 0, 0, 0, 0};  // mu.grad, ||G||^2, ||grad_+||^2, ||G-Gp||^2, ||l2-l2p||^2
  for (int r = r0 + threadIdx.x; r < r1; r += kRedThreads) {
    const double grad = a.acc[r] - (double)a.b[r];
    const double G = a.D[r] * grad;
    v[0] += (double)a.mu[r] * grad;
    v[1] += G * G;
    const double gp = fmax(grad, 0.0);
    v[2] += gp * gp;
    if (t > 0) {
      const double dg = G - a.G_prev[r], dl = a.lam2[r] - a.lam2_prev[r];
      v[3] += dg * dg;
      v[4] += dl * dl;
    }
  }
  block_sum<5>(v, sm);
  if (threadIdx.x < 5) a.part[threadIdx.x * gridDim.x + blockIdx.x] = v[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 5) {  // fixed order over the CTAs
    double q = 0.0;
    for (int c = 0; c < (int)gridDim.x; ++c) q += __ldcg(a.part + threadIdx.x * gridDim.x + c);
    sm[threadIdx.x][0] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.done = 0;
    const double gamma = st.gamma;
    const double g = a.acc[n] + a.acc[n + 1] + sm[0][0];
    const bool changed = t > 0 && gamma != st.gamma_prev;
    const double cap = st.max_step * gamma / st.gamma_ref;
    double eta;
    if (t == 0) {
      eta = st.init_step;
    } else if (changed) {
      eta = fmin(st.eta * gamma / st.gamma_prev, cap);
    } else {
      const double dl = sqrt(sm[4][0]), dg = sqrt(sm[3][0]);
      eta = (dl > 0.0 && dg > 0.0) ? fmin(dl / dg, cap) : cap;
    }
    const int64_t k = changed ? 1 : st.k;
    a.scal[0] = eta;
    a.scal[1] = (double)(k - 1) / (double)(k + 2);
    if (t < st.hist_cap) {
      dl_iter_record rec;
      rec.iter = t;
      rec.g = g;
      rec.gamma = gamma;
      rec.eta = eta;
      rec.gnorm = sqrt(sm[1][0]);
      rec.infeas = sqrt(sm[2][0]);
      rec.nnz_x = a.acc[n + 2];
      a.hist[t] = rec;
    }
    AgdDev nst = st;
    nst.gamma_prev = gamma;
    nst.gamma = gamma_at(st, t + 1);
    nst.eta = eta;
    nst.t = t + 1;
    nst.k = k + 1;
    *a.st = nst;
  }
}

// lam1' = max(lam2 + eta G, 0); lam2' = max(lam1' + beta (lam1' - lam1), 0); mu = fl32(D lam2')
__global__ void __launch_bounds__(kRedThreads) agd_update_kernel(const StepArgs a) {
  const int n = a.n;
  const double eta = a.scal[0], beta = a.scal[1];
  for (int r = blockIdx.x * kRedThreads + threadIdx.x; r < n; r += gridDim.x * kRedThreads) {
    const double grad = a.acc[r] - (double)a.b[r];
    const double G = a.D[r] * grad;
    const double l2 = a.lam2[r];
    const double l1n = fmax(l2 + eta * G, 0.0);
    const double l2n = fmax(l1n + beta * (l1n - a.lam1[r]), 0.0);
    a.G_prev[r] = G;
    a.lam2_prev[r] = l2;
    a.lam1[r] = l1n;
    a.lam2[r] = l2n;
    a.mu[r] = (float)(a.D[r] * l2n);
  }
  if (blockIdx.x == 0 && threadIdx.x < 8) a.ctr[threadIdx.x] = 0;
}

// grad = A x - b (or A x if partial), un-permuted to ORIGINAL order; obj = {g, c^T x, reg, nnz(x)}.
__global__ void __launch_bounds__(kStepThreads) finalize_kernel(const FinalizeArgs a) {
  __shared__ double sm[1][32];
  const int n = a.n;
  double v[1] = {0.0};
  for (int r = threadIdx.x; r < n; r += kStepThreads) {
    const int k = r / a.J, j = r - k * a.J;
    const int l = k * a.J + a.lab[j];
    const double g = a.partial ? a.acc[l] : a.acc[l] - (double)a.b[l];
    a.grad[r] = g;
    v[0] += (double)a.lam[l] * g;
  }
  block_sum<1>(v, sm);
  if (threadIdx.x == 0) {
    a.obj[0] = a.partial ? 0.0 : a.acc[n] + a.acc[n + 1] + v[0];
    a.obj[1] = a.acc[n];
    a.obj[2] = a.acc[n + 1];
    a.obj[3] = a.acc[n + 2];
  }
}

__global__ void row_sqnorms_kernel(const int32_t* dest, const float* a, int64_t a_stride, int64_t n, int32_t m,
                                   int32_t J, const int32_t* unlab, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = unlab[dest[e]];
    for (int f = 0; f < m; ++f) {
      const double v = (double)a[f * a_stride + e];
      if (v != 0.0) atomicAdd(out + (size_t)f * J + j, v * v);
    }
  }
}

__global__ void jacobi_diag_kernel(const double* rowsq, const int32_t* lab, double* D, int32_t m, int32_t J) {
  const int n = m * J;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int k = r / J, j = r - k * J;
    const double q = rowsq ? rowsq[r] : 0.0;
    D[k * J + lab[j]] = q > 0.0 ? 1.0 / sqrt(q) : 1.0;  // zero rows left unscaled
  }
}

__global__ void fill_kernel(double* p, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void scale_out_kernel(const double* D, const double* lam, const int32_t* lab, double* out, int32_t m,
                                 int32_t J) {
  const int n = m * J;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int k = r / J, l = k * J + lab[r - k * J];
    out[r] = D[l] * lam[l];
  }
}

__global__ void permute_f32_kernel(const float* in, const int32_t* lab, float* out, int32_t m, int32_t J, int inv) {
  const int n = m * J;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int k = r / J, l = k * J + lab[r - k * J];
    if (inv) out[r] = in[l];
    else out[l] = in[r];
  }
}

template <class T>
__global__ void relabel_gather_kernel(const T* v, T* tmp, const int32_t* unlab_old, const int32_t* lab_new, int32_t m,
                                      int32_t J) {
  const int n = m * J;  // tmp[k*J + lab_new[j]] = v[k*J + lab_old[j]], j = unlab_old[l_old]
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int k = r / J, lo = r - k * J;
    tmp[k * J + lab_new[unlab_old[lo]]] = v[r];
  }
}

__global__ void relabel_dest_kernel(int32_t* dest, int64_t n, const int32_t* unlab_old, const int32_t* lab_new) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dest[e] = lab_new[unlab_old[dest[e]]];
}

__global__ void dest_histogram_kernel(const int32_t* dest, int64_t n, int32_t J, unsigned long long* counts) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)dest[e];
    if (j < (uint32_t)J) atomicAdd(counts + j, 1ull);
  }
}

// One warp per source of [i0, i1): copy its entries from the caller's CSR chunk into the layout,
// relabelling destinations.
__global__ void build_layout_kernel(const LayoutArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = a.i0 + w0; i < a.i1; i += nw) {
    const int32_t b = a.blk_of_src[i];
    if (b < 0) continue;
    const int64_t s0 = a.row_ptr[i] - a.e0, len = a.row_ptr[i + 1] - a.row_ptr[i];
    const int64_t d0 = a.blk_off[b];
    for (int64_t e = lane; e < len; e += 32) {
      const int32_t j = a.dest[s0 + e];
      if ((uint32_t)j >= (uint32_t)a.J) {
        *a.bad = 1;
        continue;
      }
      a.dest_out[d0 + e] = a.lab[j];
      a.c_out[d0 + e] = a.c[s0 + e];
      for (int f = 0; f < a.m; ++f) a.a_out[f * a.a_stride_out + d0 + e] = a.a[f * a.a_in_stride + s0 + e];
    }
    // padding of buckets 5..8 (stored_len): label 0, c = +inf, a = 0 -> never a candidate
    const int64_t slen = (len >= 16 && len < 256) ? (len + kAlign - 1) / kAlign * kAlign : len;
    if (lane < slen - len) {
      const int64_t e = d0 + len + lane;
      a.dest_out[e] = 0;
      a.c_out[e] = __int_as_float(0x7f800000);
      for (int f = 0; f < a.m; ++f) a.a_out[f * a.a_stride_out + e] = 0.f;
    }
    if (lane == 0 && a.vsq_out) {
      const float v = a.v[i - a.i0];
      a.vsq_out[b] = v * v;
      a.vinv_out[b] = (float)(1.0 / ((double)v * (double)v));
    }
  }
}

}  // namespace

cudaError_t launch_agd_step(const StepArgs& a, cudaStream_t s) {
  const int ctas = std::max(1, std::min(kStepCtas, (a.n + kRedThreads - 1) / kRedThreads));
  agd_reduce_kernel<<<ctas, kRedThreads, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  agd_update_kernel<<<std::max(1, std::min(4 * 148, (a.n + kRedThreads - 1) / kRedThreads)), kRedThreads, 0, s>>>(a);
  return cudaGetLastError();
}
// 32 rows x 8 copy groups per CTA: warp w sums copies w, w + 8, ... of row (CTA base + lane) in
// order, warp 0 adds the 8 group sums in order; every copy row read is zeroed for the next pass.
// Loads are issued kB at a time before any store (the zeroing stores would otherwise serialise them).
__global__ void __launch_bounds__(256) partial_sum_kernel(double* part, int64_t stride, int32_t copies, int64_t n,
                                                          double* acc) {
  constexpr int kB = 10;
  __shared__ double sm[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + lane;
  double v = 0.0;
  if (r < n) {
    for (int c0 = w; c0 < copies; c0 += 8 * kB) {
      double t[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int c = c0 + 8 * k;
        t[k] = c < copies ? __ldcg(part + (size_t)c * stride + r) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int c = c0 + 8 * k;
        v += t[k];
        if (c < copies) part[(size_t)c * stride + r] = 0.0;
      }
    }
  }
  sm[w][lane] = v;
  __syncthreads();
  if (w == 0 && r < n) {
    double t = sm[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += sm[k][lane];
    acc[r] = t;
  }
}

cudaError_t launch_partial_sum(double* part, int64_t stride, int32_t copies, int64_t n, double* acc, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  partial_sum_kernel<<<(unsigned)((n + 31) / 32), 256, 0, s>>>(part, stride, copies, n, acc);
  return cudaGetLastError();
}
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
  finalize_kernel<<<1, kStepThreads, 0, s>>>(a);
  return cudaGetLastError();
}
static int grid_for(int64_t n, int64_t cap = 148 * 16) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, cap)); }
cudaError_t launch_row_sqnorms(const int32_t* dest, const float* a, int64_t a_stride, int64_t n, int32_t m,
                               int32_t J, const int32_t* unlab, double* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  row_sqnorms_kernel<<<grid_for(n), 256, 0, s>>>(dest, a, a_stride, n, m, J, unlab, out);
  return cudaGetLastError();
}
cudaError_t launch_jacobi_diag(const double* rowsq, const int32_t* lab, double* D, int32_t m, int32_t J,
                               cudaStream_t s) {
  jacobi_diag_kernel<<<grid_for((int64_t)m * J, 4096), 256, 0, s>>>(rowsq, lab, D, m, J);
  return cudaGetLastError();
}
cudaError_t launch_fill_f64(double* p, double v, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  fill_kernel<<<grid_for(n, 4096), 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}
cudaError_t launch_scale_out(const double* D, const double* lam, const int32_t* lab, double* out, int32_t m,
                             int32_t J, cudaStream_t s) {
  scale_out_kernel<<<grid_for((int64_t)m * J, 4096), 256, 0, s>>>(D, lam, lab, out, m, J);
  return cudaGetLastError();
}
cudaError_t launch_permute_f32(const float* in, const int32_t* lab, float* out, int32_t m, int32_t J, int inverse,
                               cudaStream_t s) {
  permute_f32_kernel<<<grid_for((int64_t)m * J, 4096), 256, 0, s>>>(in, lab, out, m, J, inverse);
  return cudaGetLastError();
}
cudaError_t launch_relabel_vec_f64(double* v, double* tmp, const int32_t* unlab_old, const int32_t* lab_new,
                                   int32_t m, int32_t J, cudaStream_t s) {
  relabel_gather_kernel<double><<<grid_for((int64_t)m * J, 4096), 256, 0, s>>>(v, tmp, unlab_old, lab_new, m, J);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(v, tmp, (size_t)m * J * sizeof(double), cudaMemcpyDeviceToDevice, s);
}
cudaError_t launch_relabel_vec_f32(float* v, float* tmp, const int32_t* unlab_old, const int32_t* lab_new, int32_t m,
                                   int32_t J, cudaStream_t s) {
  relabel_gather_kernel<float><<<grid_for((int64_t)m * J, 4096), 256, 0, s>>>(v, tmp, unlab_old, lab_new, m, J);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(v, tmp, (size_t)m * J * sizeof(float), cudaMemcpyDeviceToDevice, s);
}
cudaError_t launch_relabel_dest(int32_t* dest, int64_t n, const int32_t* unlab_old, const int32_t* lab_new,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  relabel_dest_kernel<<<grid_for(n, 148 * 32), 256, 0, s>>>(dest, n, unlab_old, lab_new);
  return cudaGetLastError();
}
cudaError_t launch_dest_histogram(const int32_t* dest, int64_t n, int32_t J, unsigned long long* counts,
                                  cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  dest_histogram_kernel<<<grid_for(n, 148 * 32), 256, 0, s>>>(dest, n, J, counts);
  return cudaGetLastError();
}
cudaError_t launch_build_layout(const LayoutArgs& a, cudaStream_t s) {
  if (a.i1 <= a.i0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>(((a.i1 - a.i0) * 32 + 255) / 256, 148 * 32);
  build_layout_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace dl
