// Fused dual-gradient kernels for m = 1 families, polytope kind 1 (see grad_impl.cuh).
#define DL_GRAD_M 1
#define DL_GRAD_KIND 1
#include "grad_impl.cuh"
