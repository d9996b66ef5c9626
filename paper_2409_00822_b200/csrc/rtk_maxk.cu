// rtk_maxk.cu -- MaxK-GNN consumer shapes around the row top-k.
//
// MaxK-GNN keeps the k largest entries of every hidden row
// and feeds them, as a fixed-k-per-row sparse matrix, to the aggregation
// SpMM.  The row top-k output (values[N,k], ascending int32 column indices)
// already is that layout (CSR with row_ptr = k*r).  This file adds the two
// dense <-> fixed-k conversions the layer needs around it:
//   rtk_scatter_rows_f32: dense[r, idx[r,j]] = vals[r,j], zeros elsewhere --
//     the MaxK nonlinearity's dense output and the backward of the gather;
//   rtk_gather_rows_f32:  vals[r,j] = dense[r, idx[r,j]] -- the backward of
//     the MaxK nonlinearity (gradient at the selected entries).
// Both are HBM-bound: one warp per row, the dense row staged through shared
// memory in 1024-column tiles so each output line is written once with
// 128-bit stores.  Indices outside [0, m) are ignored (scatter) / read as 0
// (gather).
#include <cuda_runtime.h>

#include <cstdint>

#include "rtk.h"

int rtk_fail(int code, const char* fmt, ...);
int rtk_device_sms();

namespace {

constexpr int kWarps = 8;        // warps per CTA
constexpr int kTile = 1024;      // dense columns staged per warp

__global__ void __launch_bounds__(kWarps * 32) scatter_rows_kernel(const float* __restrict__ vals,
                                                                   const int32_t* __restrict__ idx, int64_t ldv,
                                                                   int64_t n, int32_t k, int64_t m,
                                                                   float* __restrict__ out, int64_t ldo, bool vec) {
    __shared__ __align__(16) float tile[kWarps][kTile];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    float* t = tile[w];
    const int64_t nw = (int64_t)gridDim.x * kWarps;
    for (int64_t r = (int64_t)blockIdx.x * kWarps + w; r < n; r += nw) {
        const float* vr = vals + r * ldv;
        const int32_t* ir = idx + r * ldv;
        float* orow = out + r * ldo;
        for (int64_t c0 = 0; c0 < m; c0 += kTile) {
            const int width = (int)((m - c0) < kTile ? (m - c0) : kTile);
            for (int c = 4 * lane; c < width; c += 128) *reinterpret_cast<float4*>(t + c) = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            for (int j = lane; j < k; j += 32) {
                const int64_t col = (int64_t)ir[j] - c0;
                if (col >= 0 && col < width) t[col] = vr[j];
            }
            __syncwarp();
            if (vec) {
                for (int c = 4 * lane; c < width; c += 128)
                    *reinterpret_cast<float4*>(orow + c0 + c) = *reinterpret_cast<const float4*>(t + c);
            } else {
                for (int c = lane; c < width; c += 32) orow[c0 + c] = t[c];
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(kWarps * 32) gather_rows_kernel(const float* __restrict__ dense, int64_t ldd,
                                                                  const int32_t* __restrict__ idx, int64_t ldv,
                                                                  int64_t n, int32_t k, int64_t m,
                                                                  float* __restrict__ vals) {
    const int64_t total = n * (int64_t)k;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t r = e / k;
        const int j = (int)(e - r * k);
        const int64_t col = idx[r * ldv + j];
        vals[r * ldv + j] = (col >= 0 && col < m) ? dense[r * ldd + col] : 0.0f;
    }
}

int grid_for(int64_t items, int per_cta, int cap_per_sm) {
    int64_t g = (items + per_cta - 1) / per_cta;
    const int64_t cap = (int64_t)rtk_device_sms() * cap_per_sm;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int rtk_scatter_rows_f32(const float* vals, const int32_t* idx, int64_t ldv, int64_t n, int32_t k, int64_t m,
                         float* out, int64_t ldo, void* stream) {
    if (n < 0 || k < 1 || m < 1 || ldv < k || ldo < m) return rtk_fail(RTK_EINVAL, "bad scatter shape");
    if (n == 0) return RTK_OK;
    if (!vals || !idx || !out) return rtk_fail(RTK_EINVAL, "NULL pointer");
    const bool vec = (m % 4 == 0) && (ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    scatter_rows_kernel<<<grid_for(n, kWarps, 8), kWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(
        vals, idx, ldv, n, k, m, out, ldo, vec);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RTK_OK : rtk_fail(RTK_ECUDA, "scatter launch failed: %s", cudaGetErrorString(e));
}

int rtk_gather_rows_f32(const float* dense, int64_t ldd, const int32_t* idx, int64_t ldv, int64_t n, int32_t k,
                        int64_t m, float* vals, void* stream) {
    if (n < 0 || k < 1 || m < 1 || ldv < k || ldd < m) return rtk_fail(RTK_EINVAL, "bad gather shape");
    if (n == 0) return RTK_OK;
    if (!vals || !idx || !dense) return rtk_fail(RTK_EINVAL, "NULL pointer");
    gather_rows_kernel<<<grid_for(n * (int64_t)k, 256, 16), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        dense, ldd, idx, ldv, n, k, m, vals);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RTK_OK : rtk_fail(RTK_ECUDA, "gather launch failed: %s", cudaGetErrorString(e));
}

}  // extern "C"
