// Fused dual-gradient kernels for m = 3 families, polytope kind 0 (see grad_impl.cuh).
#define DL_GRAD_M 3
#define DL_GRAD_KIND 0
#include "grad_impl.cuh"
