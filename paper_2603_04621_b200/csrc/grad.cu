// launch_fused_grad: dispatch on (m, polytope kind) to the translation units
// grad_m<M>_k<KIND>.cu (kernels in grad_impl.cuh).
#include "internal.h"

namespace dl {

template <int M>
static cudaError_t launch_m(const GradArgs& a, int ctas, size_t smem, cudaStream_t s) {
  switch (a.kind) {
    case DL_PROJ_SIMPLEX: return launch_fused_grad_mk<M, DL_PROJ_SIMPLEX>(a, ctas, smem, s);
    case DL_PROJ_BOXCUT: return launch_fused_grad_mk<M, DL_PROJ_BOXCUT>(a, ctas, smem, s);
    case DL_PROJ_BOX: return launch_fused_grad_mk<M, DL_PROJ_BOX>(a, ctas, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fused_grad(const GradArgs& a, int ctas, size_t smem, cudaStream_t s) {
  switch (a.m) {
    case 1: return launch_m<1>(a, ctas, smem, s);
    case 2: return launch_m<2>(a, ctas, smem, s);
    case 3: return launch_m<3>(a, ctas, smem, s);
    case 4: return launch_m<4>(a, ctas, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dl
