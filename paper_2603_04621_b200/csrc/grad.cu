// launch_fused_grad: dispatch on the number of constraint families m to the per-m
// translation units grad_m1.cu .. grad_m4.cu (kernels in grad_impl.cuh).
#include "internal.h"

namespace dl {

cudaError_t launch_fused_grad(const GradArgs& a, int ctas, size_t smem, cudaStream_t s) {
  switch (a.m) {
    case 1: return launch_fused_grad_m<1>(a, ctas, smem, s);
    case 2: return launch_fused_grad_m<2>(a, ctas, smem, s);
    case 3: return launch_fused_grad_m<3>(a, ctas, smem, s);
    case 4: return launch_fused_grad_m<4>(a, ctas, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dl
