// Kernel instantiations for the cuckoo design (see ws_kernels.cuh).
#include "ws_kernels.cuh"

WS_DEFINE_DESIGN(D_CUCKOO, cuckoo)
