// Fused dual-gradient kernels for m = 3 constraint families (see grad_impl.cuh).
#define DL_GRAD_M 3
#include "grad_impl.cuh"
