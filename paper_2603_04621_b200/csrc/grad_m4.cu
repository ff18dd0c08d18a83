// Fused dual-gradient kernels for m = 4 constraint families (see grad_impl.cuh).
#define DL_GRAD_M 4
#include "grad_impl.cuh"
