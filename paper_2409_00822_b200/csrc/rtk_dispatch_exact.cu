// rtk_dispatch_exact.cu -- instantiates the exact-mode kernels (see rtk_dispatch.cuh).
#include "rtk_dispatch.cuh"

int rtk_dispatch_exact(const rtk::Args& a, cudaStream_t s) { return rtk_dispatch::dispatch<rtk::kExact>(a, s); }
int rtk_describe_exact(const rtk::Args& a, int* shape3) { return rtk_dispatch::describe_dispatch<rtk::kExact>(a, shape3); }
