// Fused dual-gradient kernels for m = 3 families, polytope kind 1 (see grad_impl.cuh).
#define DL_GRAD_M 3
#define DL_GRAD_KIND 1
#include "grad_impl.cuh"
