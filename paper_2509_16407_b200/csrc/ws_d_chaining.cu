// Kernel instantiations for the chaining design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_CHAINING, chaining)
