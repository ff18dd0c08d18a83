// Fused dual-gradient kernels for m = 2 constraint families (see grad_impl.cuh).
#define DL_GRAD_M 2
#include "grad_impl.cuh"
