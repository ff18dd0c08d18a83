// Small kernels around the fused pass: AGD step (K2), gradient finalize (K3),
// Jacobi row norms (K4), layout build (K5).
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

#include "internal.h"

namespace dl {
namespace {

constexpr int kStepThreads = 1024;

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

template <int NV>
__device__ void block_max(float (&v)[NV], float (*sm)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    for (int o = 16; o > 0; o >>= 1) v[i] = fmaxf(v[i], __shfl_xor_sync(0xffffffffu, v[i], o));
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sm[i][warp] = v[i];
  __syncthreads();
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float t = 0.f;
    for (int w = 0; w < nw; ++w) t = fmaxf(t, sm[i][w]);
    v[i] = t;
  }
  __syncthreads();
}

// fl32 error bound of the fused kernel's s = fl(c + sum a lambda): 2^-19 (m+1) magnitude bound
__device__ __forceinline__ float slack_of(int m, float cmax, const float* amax, const float* lmax) {
  float B = cmax;
  for (int f = 0; f < m; ++f) B += amax[f] * lmax[f];
  return 1.9073486e-6f * (float)(m + 1) * B * 1.0001f;
}

__device__ __forceinline__ double gamma_at(const AgdDev& st, int64_t t) {
  if (!st.continuation) return st.gamma0;
  int64_t h = t / st.halve_every;
  double g = h > 2000 ? 0.0 : ldexp(st.gamma0, -(int)h);
  return fmax(g, st.gamma_min);
}

// One AGD iteration (R5-R8; oracle/agd.py steps 2-5) from the accumulated
// A x*(mu_t) (+ objective scalars).  Single CTA => every rank computes identical bits.
__global__ void __launch_bounds__(kStepThreads) agd_step_kernel(const StepArgs a) {
  __shared__ double sm[6][32];
  __shared__ double s_eta, s_beta;
  const int n = a.n;
  const AgdDev st = *a.st;
  const int64_t t = st.t;
  const double gamma = st.gamma;
  // pass 1: dual value and norms
  double v[5] = {0, 0, 0, 0, 0};  // mu.grad, ||G||^2, ||grad_+||^2, ||G-Gp||^2, ||l2-l2p||^2
  for (int r = threadIdx.x; r < n; r += kStepThreads) {
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
  if (threadIdx.x == 0) {
    const double g = a.acc[n] + a.acc[n + 1] + v[0];
    const bool changed = t > 0 && gamma != st.gamma_prev;
    const double cap = st.max_step * gamma / st.gamma_ref;
    double eta;
    if (t == 0) {
      eta = st.init_step;
    } else if (changed) {
      eta = fmin(st.eta * gamma / st.gamma_prev, cap);
    } else {
      const double dl = sqrt(v[4]), dg = sqrt(v[3]);
      eta = (dl > 0.0 && dg > 0.0) ? fmin(dl / dg, cap) : cap;
    }
    const int64_t k = changed ? 1 : st.k;
    s_eta = eta;
    s_beta = (double)(k - 1) / (double)(k + 2);
    if (t < st.hist_cap) {
      dl_iter_record rec;
      rec.iter = t;
      rec.g = g;
      rec.gamma = gamma;
      rec.eta = eta;
      rec.gnorm = sqrt(v[1]);
      rec.infeas = sqrt(v[2]);
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
  __syncthreads();
  const double eta = s_eta, beta = s_beta;
  // pass 2: lam1' = max(lam2 + eta G, 0); lam2' = max(lam1' + beta (lam1' - lam1), 0)
  float lmax[4] = {0.f, 0.f, 0.f, 0.f};
  const int J = n / a.m;
  for (int r = threadIdx.x; r < n; r += kStepThreads) {
    const double grad = a.acc[r] - (double)a.b[r];
    const double G = a.D[r] * grad;
    const double l2 = a.lam2[r];
    const double l1n = fmax(l2 + eta * G, 0.0);
    const double l2n = fmax(l1n + beta * (l1n - a.lam1[r]), 0.0);
    a.G_prev[r] = G;
    a.lam2_prev[r] = l2;
    a.lam1[r] = l1n;
    a.lam2[r] = l2n;
    const float mu = (float)(a.D[r] * l2n);
    a.mu[r] = mu;
    const int f = r / J;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q == f) lmax[q] = fmaxf(lmax[q], fabsf(mu));
    a.acc[r] = 0.0;
  }
  if (threadIdx.x < 4) a.acc[n + threadIdx.x] = 0.0;
  if (threadIdx.x < 8) a.ctr[threadIdx.x] = 0;
  __shared__ float smx[4][32];
  block_max<4>(lmax, smx);
  if (threadIdx.x == 0) *a.slack = slack_of(a.m, a.cmax, a.amax, lmax);
}

__global__ void __launch_bounds__(kStepThreads) slack_kernel(const float* lam, int32_t m, int32_t J, float cmax,
                                                             float a0, float a1, float a2, float a3, float* out) {
  __shared__ float smx[4][32];
  float lmax[4] = {0.f, 0.f, 0.f, 0.f};
  for (int f = 0; f < m; ++f)
    for (int j = threadIdx.x; j < J; j += kStepThreads) lmax[f] = fmaxf(lmax[f], fabsf(lam[(size_t)f * J + j]));
  block_max<4>(lmax, smx);
  const float amax[4] = {a0, a1, a2, a3};
  if (threadIdx.x == 0) *out = slack_of(m, cmax, amax, lmax);
}

__global__ void absmax_kernel(const float* x, int64_t n, unsigned int* out) {
  float v = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (fabsf(x[i]) < __int_as_float(0x7f800000)) v = fmaxf(v, fabsf(x[i]));  // layout padding is +inf
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(v));  // v >= 0: uint order = float order
}

// grad = A x - b (or A x if partial); obj = {g, c^T x, reg, nnz(x)}.
__global__ void __launch_bounds__(kStepThreads) finalize_kernel(const FinalizeArgs a) {
  __shared__ double sm[1][32];
  const int n = a.n;
  double v[1] = {0.0};
  for (int r = threadIdx.x; r < n; r += kStepThreads) {
    const double g = a.partial ? a.acc[r] : a.acc[r] - (double)a.b[r];
    a.grad[r] = g;
    v[0] += (double)a.lam[r] * g;
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
                                   int32_t J, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = dest[e];
    for (int f = 0; f < m; ++f) {
      const double v = (double)a[f * a_stride + e];
      if (v != 0.0) atomicAdd(out + (size_t)f * J + j, v * v);
    }
  }
}

__global__ void jacobi_diag_kernel(const double* rowsq, double* D, int32_t n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double q = rowsq ? rowsq[r] : 0.0;
    D[r] = q > 0.0 ? 1.0 / sqrt(q) : 1.0;  // zero rows left unscaled
  }
}

__global__ void fill_kernel(double* p, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void scale_out_kernel(const double* D, const double* lam, double* out, int32_t n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) out[r] = D[r] * lam[r];
}

// One warp per block: copy its entries from the caller's CSR into the layout.
__global__ void build_layout_kernel(const LayoutArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w0; b < a.num_blocks; b += nw) {
    const int64_t i = a.perm[b];
    const int64_t s0 = a.row_ptr[i], len = a.row_ptr[i + 1] - s0;
    const int64_t d0 = a.blk_off[b];
    for (int64_t e = lane; e < len; e += 32) {
      const int32_t j = a.dest[s0 + e];
      if ((uint32_t)j >= (uint32_t)a.J) *a.bad = 1;
      a.dest_out[d0 + e] = j;
      a.c_out[d0 + e] = a.c[s0 + e];
      for (int f = 0; f < a.m; ++f) a.a_out[f * a.a_stride_out + d0 + e] = a.a[f * a.nnz + s0 + e];
    }

    if (lane == 0 && a.vsq_out) {
      const float v = a.v[i];
      a.vsq_out[b] = v * v;
      a.vinv_out[b] = (float)(1.0 / ((double)v * (double)v));
    }
  }
}

}  // namespace

cudaError_t launch_agd_step(const StepArgs& a, cudaStream_t s) {
  agd_step_kernel<<<1, kStepThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_absmax(const float* x, int64_t n, float* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float), s);
  if (e != cudaSuccess || n == 0) return e;
  absmax_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(x, n,
                                                                                 reinterpret_cast<unsigned int*>(out));
  return cudaGetLastError();
}
cudaError_t launch_slack(const float* lam, int32_t m, int32_t J, float cmax, const float* amax4, float* out,
                         cudaStream_t s) {
  slack_kernel<<<1, kStepThreads, 0, s>>>(lam, m, J, cmax, amax4[0], amax4[1], amax4[2], amax4[3], out);
  return cudaGetLastError();
}
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
  finalize_kernel<<<1, kStepThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_row_sqnorms(const int32_t* dest, const float* a, int64_t a_stride, int64_t n, int32_t m,
                               int32_t J, double* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  row_sqnorms_kernel<<<blocks, 256, 0, s>>>(dest, a, a_stride, n, m, J, out);
  return cudaGetLastError();
}
cudaError_t launch_jacobi_diag(const double* rowsq, double* D, int32_t n, cudaStream_t s) {
  jacobi_diag_kernel<<<(n + 255) / 256, 256, 0, s>>>(rowsq, D, n);
  return cudaGetLastError();
}
cudaError_t launch_fill_f64(double* p, double v, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  fill_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}
cudaError_t launch_scale_out(const double* D, const double* lam, double* out, int32_t n, cudaStream_t s) {
  scale_out_kernel<<<(n + 255) / 256, 256, 0, s>>>(D, lam, out, n);
  return cudaGetLastError();
}
cudaError_t launch_build_layout(const LayoutArgs& a, cudaStream_t s) {
  if (a.num_blocks == 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((a.num_blocks * 32 + 255) / 256, 148 * 32);
  build_layout_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace dl
