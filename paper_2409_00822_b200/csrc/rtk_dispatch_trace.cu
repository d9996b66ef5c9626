// rtk_dispatch_trace.cu -- instantiates the trace-mode kernels (see rtk_dispatch.cuh).
#include "rtk_dispatch.cuh"

int rtk_dispatch_trace(const rtk::Args& a, cudaStream_t s) { return rtk_dispatch::dispatch<rtk::kTrace>(a, s); }
int rtk_describe_trace(const rtk::Args& a, int* shape3) { return rtk_dispatch::describe_dispatch<rtk::kTrace>(a, shape3); }
