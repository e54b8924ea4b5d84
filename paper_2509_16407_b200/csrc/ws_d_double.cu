// Kernel instantiations for the double design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_DOUBLE, double)
