// Kernel instantiations for the iceberg_md design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_ICEBERG_MD, iceberg_md)
