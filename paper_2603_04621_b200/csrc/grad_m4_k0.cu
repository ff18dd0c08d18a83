// Fused dual-gradient kernels for m = 4 families, polytope kind 0 (see grad_impl.cuh).
#define DL_GRAD_M 4
#define DL_GRAD_KIND 0
#include "grad_impl.cuh"
