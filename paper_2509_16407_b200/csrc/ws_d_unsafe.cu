// Kernel instantiations for the unsafe design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_UNSAFE, unsafe)
