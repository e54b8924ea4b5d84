// Kernel instantiations for the iceberg design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_ICEBERG, iceberg)
