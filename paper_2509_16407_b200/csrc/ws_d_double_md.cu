// Kernel instantiations for the double_md design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_DOUBLE_MD, double_md)
