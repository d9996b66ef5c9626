// rtk_dispatch_early.cu -- instantiates the early-mode kernels (see rtk_dispatch.cuh).
#include "rtk_dispatch.cuh"

int rtk_dispatch_early(const rtk::Args& a, cudaStream_t s) { return rtk_dispatch::dispatch<rtk::kEarly>(a, s); }
int rtk_describe_early(const rtk::Args& a, int* shape3) { return rtk_dispatch::describe_dispatch<rtk::kEarly>(a, shape3); }
