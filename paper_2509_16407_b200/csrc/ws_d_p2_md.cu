// Kernel instantiations for the p2_md design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_P2_MD, p2_md)
