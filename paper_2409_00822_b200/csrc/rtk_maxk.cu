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
// And the aggregation that consumes the fixed-k rows (MaxK-GNN's SpMM with
// the top-k-processed right-hand matrix):
//   rtk_maxk_spmm_f32: out[i, :] = sum over edges e = (i, j) of a_e * H_j,
//     H_j the fixed-k row j (vals[j, :] at columns idx[j, :], int32 or uint8);
//   rtk_maxk_spmm_backward_f32: grad_vals[j, t] = sum over edges (i, j) of
//     a_e * grad_out[i, idx[j, t]] (over the transposed graph's CSR).
// Per edge only the k (value, column) pairs of row j are read (k*(4+4) or
// k*(4+1) bytes instead of the dense row's 4*m), which is MaxK-GNN's point.
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


constexpr int kSpmmWarps = 8;  // warps per CTA of the aggregation kernels
constexpr int kSpmmMaxM = 1024;

// Index of entry t of fixed-k row j: int32 or uint8 storage.
__device__ __forceinline__ int fixed_col(const int32_t* __restrict__ idx, const uint8_t* __restrict__ idx8,
                                         int64_t off) {
    return idx8 ? (int)idx8[off] : (int)idx[off];
}

// One warp per output row i; the m-float accumulator lives in the warp's
// shared-memory row.  Edges are taken 32 at a time (lane l loads edge
// e0 + l's column and weight, broadcast by SHFL); four edges' (value,
// column) loads are issued before their updates to overlap the L2 latency.
// Lane t < k adds a_e * vals[j, t] into column idx[j, t] with a shared-memory
// read-modify-write (one FFMA): a row's k columns are distinct, so the lanes
// of one edge never collide, and a __syncwarp between edges orders the
// updates -- every column sums its terms in edge order, deterministically.
// (A shared RED.ADD per entry measured 20% slower.)  IdxT: int32_t or
// uint8_t columns; offsets are 32-bit (the host checks n_in * ldv < 2^31).
template <class IdxT>
__global__ void __launch_bounds__(kSpmmWarps * 32) maxk_spmm_kernel(
    const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const float* __restrict__ aval, int64_t n,
    const float* __restrict__ vals, const IdxT* __restrict__ idx, unsigned ldv, int32_t k, int32_t m,
    float* __restrict__ out, int64_t ldo) {
    __shared__ __align__(16) float acc_s[kSpmmWarps][kSpmmMaxM];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    float* acc = acc_s[w];
    const bool check_col = sizeof(IdxT) == 4 || m < 256;  // uint8 columns of 256-wide rows are always in range
    const int64_t nw = (int64_t)gridDim.x * kSpmmWarps;
    for (int64_t i = (int64_t)blockIdx.x * kSpmmWarps + w; i < n; i += nw) {
        for (int c = lane; c < m; c += 32) acc[c] = 0.0f;
        __syncwarp();
        const int64_t e_beg = rp[i], e_end = rp[i + 1];
        for (int64_t e0 = e_beg; e0 < e_end; e0 += 32) {
            const int ne = (int)((e_end - e0) < 32 ? (e_end - e0) : 32);
            unsigned jl = 0;
            float al = 0.0f;
            if (lane < ne) {
                jl = (unsigned)col[e0 + lane] * ldv;
                al = aval ? aval[e0 + lane] : 1.0f;
            }
            for (int u0 = 0; u0 < ne; u0 += 4) {
                float v[4], a4[4];
                int c[4];
                unsigned jo[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    jo[u] = __shfl_sync(0xffffffffu, jl, (u0 + u) & 31);
                    a4[u] = __shfl_sync(0xffffffffu, al, (u0 + u) & 31);
                    const bool on = u0 + u < ne && lane < k;
                    v[u] = on ? vals[jo[u] + lane] : 0.0f;
                    c[u] = on ? (int)idx[jo[u] + lane] : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (c[u] >= 0 && (!check_col || c[u] < m)) acc[c[u]] = __fmaf_rn(a4[u], v[u], acc[c[u]]);
                    __syncwarp();
                }
                // k > 32: the remaining entries of the same four rows (deterministic order)
                for (int t = lane + 32; t < k; t += 32) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (u0 + u >= ne) break;
                        const int cc = (int)idx[jo[u] + t];
                        if (!check_col || cc < m) acc[cc] = __fmaf_rn(a4[u], vals[jo[u] + t], acc[cc]);
                        __syncwarp(__activemask());
                    }
                }
                __syncwarp();  // lanes that skipped the loop above wait for its updates (racecheck)
            }
        }
        __syncwarp();
        float* orow = out + i * ldo;
        for (int c = lane; c < m; c += 32) orow[c] = acc[c];
        __syncwarp();
    }
}

// Backward: one warp per row j of the fixed-k matrix, lane t owns entry t
// and accumulates a_e * grad_out[i, idx[j, t]] over the in-edges of j in
// registers (edge order, deterministic).
__global__ void __launch_bounds__(kSpmmWarps * 32) maxk_spmm_backward_kernel(
    const int64_t* __restrict__ rpt, const int32_t* __restrict__ colt, const float* __restrict__ avalt, int64_t n,
    const float* __restrict__ gout, int64_t ldg, const int32_t* __restrict__ idx, const uint8_t* __restrict__ idx8,
    int64_t ldv, int32_t k, int32_t m, float* __restrict__ gvals) {
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * kSpmmWarps;
    for (int64_t j = (int64_t)blockIdx.x * kSpmmWarps + w; j < n; j += nw) {
        const int64_t e_beg = rpt[j], e_end = rpt[j + 1];
        for (int t0 = 0; t0 < k; t0 += 32) {
            const int t = t0 + lane;
            const int cc = t < k ? fixed_col(idx, idx8, j * ldv + t) : 0;
            const bool ok = t < k && (unsigned)cc < (unsigned)m;
            float g = 0.0f;
            for (int64_t e0 = e_beg; e0 < e_end; e0 += 32) {
                const int ne = (int)((e_end - e0) < 32 ? (e_end - e0) : 32);
                int il = 0;
                float al = 0.0f;
                if (lane < ne) {
                    il = colt[e0 + lane];
                    al = avalt ? avalt[e0 + lane] : 1.0f;
                }
                for (int u0 = 0; u0 < ne; u0 += 4) {  // four gathers in flight, summed in edge order
                    float gv[4], a4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t ii = __shfl_sync(0xffffffffu, il, (u0 + u) & 31);
                        a4[u] = __shfl_sync(0xffffffffu, al, (u0 + u) & 31);
                        gv[u] = (ok && u0 + u < ne) ? gout[ii * ldg + cc] : 0.0f;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (u0 + u < ne) g = __fadd_rn(g, __fmul_rn(a4[u], gv[u]));
                }
            }
            if (t < k) gvals[j * ldv + t] = g;
        }
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

int rtk_maxk_spmm_f32(const int64_t* row_ptr, const int32_t* col, const float* aval, int64_t n, const float* vals,
                      const int32_t* idx, const uint8_t* idx8, int64_t ldv, int32_t k, int64_t m, int64_t n_in,
                      float* out, int64_t ldo, void* stream) {
    if (n < 0 || k < 1 || m < 1 || m > kSpmmMaxM || ldv < k || ldo < m)
        return rtk_fail(RTK_EINVAL, "bad maxk_spmm shape (n=%lld, k=%d, m=%lld: m <= %d)", (long long)n, k,
                        (long long)m, kSpmmMaxM);
    if ((idx != nullptr) == (idx8 != nullptr)) return rtk_fail(RTK_EINVAL, "exactly one of idx / idx8 must be given");
    if (idx8 && m > 256) return rtk_fail(RTK_EINVAL, "uint8 indices need m <= 256, got %lld", (long long)m);
    if (n_in < 0 || n_in * ldv >= (1LL << 31))
        return rtk_fail(RTK_EINVAL, "fixed-k matrix too large: n_in * ldv must be < 2^31");
    if (n == 0) return RTK_OK;
    if (!row_ptr || !col || !vals || !out) return rtk_fail(RTK_EINVAL, "NULL pointer");
    const dim3 grid(grid_for(n, kSpmmWarps, 8)), block(kSpmmWarps * 32);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (idx8)
        maxk_spmm_kernel<uint8_t><<<grid, block, 0, s>>>(row_ptr, col, aval, n, vals, idx8, (unsigned)ldv, k,
                                                         (int32_t)m, out, ldo);
    else
        maxk_spmm_kernel<int32_t><<<grid, block, 0, s>>>(row_ptr, col, aval, n, vals, idx, (unsigned)ldv, k,
                                                         (int32_t)m, out, ldo);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RTK_OK : rtk_fail(RTK_ECUDA, "maxk_spmm launch failed: %s", cudaGetErrorString(e));
}

int rtk_maxk_spmm_backward_f32(const int64_t* row_ptr_t, const int32_t* col_t, const float* aval_t, int64_t n,
                               const float* grad_out, int64_t ldg, const int32_t* idx, const uint8_t* idx8,
                               int64_t ldv, int32_t k, int64_t m, float* grad_vals, void* stream) {
    if (n < 0 || k < 1 || m < 1 || ldv < k || ldg < m) return rtk_fail(RTK_EINVAL, "bad maxk_spmm_backward shape");
    if ((idx != nullptr) == (idx8 != nullptr)) return rtk_fail(RTK_EINVAL, "exactly one of idx / idx8 must be given");
    if (idx8 && m > 256) return rtk_fail(RTK_EINVAL, "uint8 indices need m <= 256, got %lld", (long long)m);
    if (n == 0) return RTK_OK;
    if (!row_ptr_t || !col_t || !grad_out || !grad_vals) return rtk_fail(RTK_EINVAL, "NULL pointer");
    maxk_spmm_backward_kernel<<<grid_for(n, kSpmmWarps, 8), kSpmmWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(
        row_ptr_t, col_t, aval_t, n, grad_out, ldg, idx, idx8, ldv, k, (int32_t)m, grad_vals);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RTK_OK
                            : rtk_fail(RTK_ECUDA, "maxk_spmm_backward launch failed: %s", cudaGetErrorString(e));
}

}  // extern "C"
