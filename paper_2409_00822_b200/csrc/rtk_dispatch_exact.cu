// rtk_dispatch_exact.cu -- instantiates the exact-mode kernels (see rtk_dispatch.cuh).
#include "rtk_dispatch.cuh"

int rtk_dispatch_exact(const rtk::Args& a, cudaStream_t s) { return rtk_dispatch::dispatch<rtk::kExact>(a, s); }
