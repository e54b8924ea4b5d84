// Kernel instantiations for the p2 design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_P2, p2)
