// Fused dual-gradient kernels for m = 1 constraint families (see grad_impl.cuh).
#define DL_GRAD_M 1
#include "grad_impl.cuh"
