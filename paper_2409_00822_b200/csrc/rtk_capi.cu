// rtk_capi.cu -- extern "C" entry points of librtk.so (declared in include/rtk.h).
//
// Host-side dispatch: validate sizes, pick the register-tile instantiation
// for (M, alignment), size the persistent grid from the occupancy of that
// instantiation (cached per device), and launch on the caller's stream.  No
// allocation, no synchronisation.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <map>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "rtk.h"
#define RTK_DEFINE_FLAT_KERNELS
#include "rtk_dispatch.cuh"

namespace {

thread_local char g_err[512] = "";

}  // namespace

// Library-internal (hidden): record the thread-local error message.
int rtk_fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

namespace {

template <class... T>
int fail(int code, const char* fmt, T... args) {
    return rtk_fail(code, fmt, args...);
}

constexpr int kFlatThreads = 256;  // threads per CTA of the elementwise kernels
constexpr int kMaxDevices = 64;

struct DeviceInfo {
    std::once_flag once;
    int sms = 0;
};
DeviceInfo g_dev[kMaxDevices];

int device_sms() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
    DeviceInfo& d = g_dev[dev];
    std::call_once(d.once, [&] {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        d.sms = v;
    });
    return d.sms;
}

// Occupancy (CTAs per SM) of one kernel instantiation at a dynamic shared
// memory size, cached per (device, kernel, smem, threads).  Kernels needing
// more than 48 KB of dynamic shared memory are opted in to the largest size
// requested so far (never lowered, so every cached size stays launchable).
std::mutex g_occ_mu;
std::map<std::tuple<int, const void*, size_t>, int> g_occ;
std::map<std::pair<int, const void*>, size_t> g_smem_optin;

int ctas_per_sm(const void* kernel, size_t smem, int threads) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto key = std::make_tuple(dev, kernel, smem + ((size_t)threads << 40));
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    if (smem > 48 * 1024) {
        size_t& cur = g_smem_optin[std::make_pair(dev, kernel)];
        if (smem > cur) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cur = smem;
        }
    }
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, smem) != cudaSuccess || blocks < 1)
        blocks = 1;
    g_occ[key] = blocks;
    return blocks;
}

int launch_flat(void (*kernel)(rtk::Args), const rtk::Args& a, cudaStream_t s, int per_item = 1) {
    const long long total = a.n * (long long)a.m / per_item;
    long long grid = (total + kFlatThreads - 1) / kFlatThreads;
    const long long cap = (long long)device_sms() * 8;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    kernel<<<(unsigned)grid, kFlatThreads, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

int check_common(const float* x, int64_t n, int64_t m, int64_t ldx) {
    if (n < 0) return fail(RTK_EINVAL, "n must be >= 0, got %lld", (long long)n);
    if (m < 1 || m > 0x7fffffff) return fail(RTK_EINVAL, "m must be in [1, 2^31), got %lld", (long long)m);
    if (n >= 0xffffffffLL) return fail(RTK_EINVAL, "n must be < 2^32 - 1, got %lld", (long long)n);
    if (ldx < m) return fail(RTK_EINVAL, "ldx (%lld) < m (%lld)", (long long)ldx, (long long)m);
    if (ldx >= (1LL << 30)) return fail(RTK_EINVAL, "ldx must be < 2^30, got %lld", (long long)ldx);
    if (n > 0 && !x) return fail(RTK_EINVAL, "x is NULL");
    return RTK_OK;
}

int reset_nan(uint32_t* nan_first_row, cudaStream_t s) {
    if (!nan_first_row) return RTK_OK;
    cudaError_t e = cudaMemsetAsync(nan_first_row, 0xff, sizeof(uint32_t), s);
    if (e != cudaSuccess) return fail(RTK_ECUDA, "cudaMemsetAsync failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

rtk::Args make_args(const float* x, int64_t n, int64_t m, int64_t ldx, int32_t k, float* vals, int32_t* idx,
                    int64_t ldo, int32_t* iters, int8_t* reasons, uint32_t* nan_first_row) {
    rtk::Args a;
    a.x = x;
    a.n = n;
    a.m = (int)m;
    a.ldx = ldx;
    a.k = k;
    a.eps_rel = 0.0;
    a.hard_cap = 64;
    a.max_iter = 4;
    a.vals = vals;
    a.idx = idx;
    a.ldo = ldo;
    a.iters = iters;
    a.reasons = reinterpret_cast<signed char*>(reasons);
    a.nan_row = nan_first_row;
    a.opaque_zero = 0;
    a.dense = nullptr;
    a.ldd = 0;
    a.idx8 = nullptr;
    a.ld8 = 0;
    a.out_vec4 = vals && idx && ((reinterpret_cast<uintptr_t>(vals) | reinterpret_cast<uintptr_t>(idx)) & 15) == 0 &&
                 ldo % 4 == 0 && k % 4 == 0 && k >= 128;  // k = 64: one half-idle iteration measured slower
    return a;
}

int rowtopk_common(int mode, const float* x, int64_t n, int64_t m, int64_t ldx, int32_t k, double eps_rel,
                   int32_t hard_cap, int32_t max_iter, float* vals, int32_t* idx, int64_t ldo, int32_t* iters,
                   int8_t* reasons, uint32_t* nan_first_row, void* stream) {
    int rc = check_common(x, n, m, ldx);
    if (rc) return rc;
    if (k < 1 || k > m) return fail(RTK_EINVAL, "k must be in [1, %lld], got %d", (long long)m, k);
    if (mode != rtk::kTrace) {
        if (ldo < k) return fail(RTK_EINVAL, "ldo (%lld) < k (%d)", (long long)ldo, k);
        if (ldo >= (1LL << 30)) return fail(RTK_EINVAL, "ldo must be < 2^30, got %lld", (long long)ldo);
        if (n > 0 && (!vals || !idx)) return fail(RTK_EINVAL, "vals/idx is NULL");
    } else if (n > 0 && (!iters || !reasons)) {
        return fail(RTK_EINVAL, "iters/reasons are required for the trace kernel");
    }
    if (mode == rtk::kExact || mode == rtk::kTrace) {
        if (!(eps_rel >= 0.0)) return fail(RTK_EINVAL, "eps_rel must be >= 0, got %g", eps_rel);
        if (hard_cap < 1) return fail(RTK_EINVAL, "hard_cap must be >= 1, got %d", hard_cap);
    } else if (max_iter < 1) {
        return fail(RTK_EINVAL, "max_iter must be >= 1, got %d", max_iter);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rc = reset_nan(nan_first_row, s);
    if (rc || n == 0) return rc;
    rtk::Args a = make_args(x, n, m, ldx, k, mode == rtk::kTrace ? nullptr : vals,
                            mode == rtk::kTrace ? nullptr : idx, ldo, iters, reasons, nan_first_row);
    a.eps_rel = eps_rel;
    a.hard_cap = hard_cap;
    a.max_iter = max_iter;
    if (k == m) {  // _kernels.py:173-179
        const bool vec = m % 4 == 0 && ldx % 4 == 0 && (!vals || ldo % 4 == 0) &&
                         ((uintptr_t)x & 15u) == 0 && ((uintptr_t)vals & 15u) == 0 && ((uintptr_t)idx & 15u) == 0 &&
                         n * (m / 4) < 0xffffffffLL;
        return launch_flat(vec ? rtk::full_copy_vec4_kernel : rtk::full_copy_kernel, a, s, vec ? 4 : 1);
    }
    switch (mode) {
        case rtk::kExact: return rtk_dispatch_exact(a, s);
        case rtk::kEarly: return rtk_dispatch_early(a, s);
        default: return rtk_dispatch_trace(a, s);
    }
}

}  // namespace

int rtk_device_sms() { return device_sms(); }

// Tensor map of x viewed as [n][32][e] floats (row stride ldx), box = one row,
// swizzle matching the row width (128B for e = 32, 64B for e = 16).  The
// driver entry point is fetched once through the runtime (no -lcuda).
// cuTensorMapEncodeTiled through the runtime's driver entry point (resolved once)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    return encode;
}

bool rtk_encode_row_map(CUtensorMap* map, const float* x, long long n, int e, long long ldx) {
    const PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode || (reinterpret_cast<uintptr_t>(x) & 15) || (ldx * 4) % 16) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)e, 32, (cuuint64_t)n};
    const cuuint64_t strides[2] = {(cuuint64_t)e * 4, (cuuint64_t)ldx * 4};
    const cuuint32_t box[3] = {(cuuint32_t)e, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                              e == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
// Lane rows of E floats as [n][32][E] split into parts of 16 / 8 / 4 floats
// (TmaRow): part p covers elements first(p) .. first(p) + widths[p] of every
// lane, 64B / 32B / no swizzle.
bool rtk_encode_row_parts(CUtensorMap* maps, const float* x, long long n, int e, long long ldx, const int* widths,
                          int parts) {
    const PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode || (reinterpret_cast<uintptr_t>(x) & 15) || (ldx * 4) % 16 || (e * 4) % 16) return false;
    const cuuint64_t strides[2] = {(cuuint64_t)e * 4, (cuuint64_t)ldx * 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    int first = 0;
    for (int p = 0; p < parts; ++p) {
        const int w = widths[p];
        const cuuint64_t dims[3] = {(cuuint64_t)w, 32, (cuuint64_t)n};
        const cuuint32_t box[3] = {(cuuint32_t)w, 32, 1};
        const CUtensorMapSwizzle sw =
            w == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : (w == 8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE);
        if (encode(&maps[p], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x + first), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        first += w;
    }
    return true;
}
int rtk_ctas_per_sm(const void* kernel, size_t smem, int threads) { return ctas_per_sm(kernel, smem, threads); }

extern "C" {

int rtk_rowtopk_exact_f32(const float* x, int64_t n, int64_t m, int64_t ldx, int32_t k, double eps_rel,
                          int32_t hard_cap, float* vals, int32_t* idx, int64_t ldo, int32_t* iters, int8_t* reasons,
                          uint32_t* nan_first_row, void* stream) {
    return rowtopk_common(rtk::kExact, x, n, m, ldx, k, eps_rel, hard_cap, 1, vals, idx, ldo, iters, reasons,
                          nan_first_row, stream);
}

int rtk_rowtopk_early_f32(const float* x, int64_t n, int64_t m, int64_t ldx, int32_t k, int32_t max_iter,
                          float* vals, int32_t* idx, int64_t ldo, int32_t* iters, int8_t* reasons,
                          uint32_t* nan_first_row, void* stream) {
    return rowtopk_common(rtk::kEarly, x, n, m, ldx, k, 0.0, 1, max_iter, vals, idx, ldo, iters, reasons,
                          nan_first_row, stream);
}

int rtk_rowtopk_x16(const void* x, int32_t dtype, int32_t mode, int64_t n, int64_t m, int64_t ldx, int32_t k,
                    int32_t hard_cap, int32_t max_iter, float* vals, int32_t* idx, int64_t ldo,
                    uint32_t* nan_first_row, void* stream) {
    if (dtype != 1 && dtype != 2) return fail(RTK_EINVAL, "dtype must be 1 (bfloat16) or 2 (float16), got %d", dtype);
    if (mode != rtk::kExact && mode != rtk::kEarly) return fail(RTK_EINVAL, "mode must be 0 or 1, got %d", mode);
    int rc = check_common(static_cast<const float*>(x), n, m, ldx);
    if (rc) return rc;
    if (k < 1 || k > m) return fail(RTK_EINVAL, "k must be in [1, %lld], got %d", (long long)m, k);
    if (ldo < k) return fail(RTK_EINVAL, "ldo (%lld) < k (%d)", (long long)ldo, k);
    if (ldo >= (1LL << 30)) return fail(RTK_EINVAL, "ldo must be < 2^30, got %lld", (long long)ldo);
    if (n > 0 && (!vals || !idx)) return fail(RTK_EINVAL, "vals/idx is NULL");
    if (mode == rtk::kExact && hard_cap < 1) return fail(RTK_EINVAL, "hard_cap must be >= 1, got %d", hard_cap);
    if (mode == rtk::kEarly && max_iter < 1) return fail(RTK_EINVAL, "max_iter must be >= 1, got %d", max_iter);
    const uintptr_t xa = reinterpret_cast<uintptr_t>(x);
    const bool pair_ok = m <= 256 && m % 4 == 0 && ldx % 4 == 0 && (xa & 7) == 0 && n < 0xffff0000LL;
    const bool long_ok = m > 256 && m <= 4096 && m % 8 == 0 && ldx % 8 == 0 && (xa & 15) == 0;
    if (k == m || !(pair_ok || long_ok))
        return fail(RTK_EUNSUPPORTED, "shape outside the native 16-bit path (m=%lld, k=%d, ldx=%lld)",
                    (long long)m, k, (long long)ldx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rc = reset_nan(nan_first_row, s);
    if (rc || n == 0) return rc;
    rtk::Args a = make_args(static_cast<const float*>(x), n, m, ldx, k, vals, idx, ldo, nullptr, nullptr,
                            nan_first_row);
    a.hard_cap = hard_cap;
    a.max_iter = max_iter;
    return rtk_dispatch_x16(a, dtype, mode, s);
}

int rtk_maxk_dense(const void* x, int32_t dtype, int32_t mode, int64_t n, int64_t m, int64_t ldx, int32_t k,
                   int32_t hard_cap, int32_t max_iter, float* vals, int32_t* idx, int64_t ldo, void* dense,
                   int64_t ldd, uint8_t* idx8, int64_t ld8, uint32_t* nan_first_row, void* stream) {
    if (dtype < 0 || dtype > 2) return fail(RTK_EINVAL, "dtype must be 0 (float32), 1 (bfloat16) or 2 (float16), got %d", dtype);
    if (mode != rtk::kExact && mode != rtk::kEarly) return fail(RTK_EINVAL, "mode must be 0 or 1, got %d", mode);
    int rc = check_common(static_cast<const float*>(x), n, m, ldx);
    if (rc) return rc;
    if (k < 1 || k > m) return fail(RTK_EINVAL, "k must be in [1, %lld], got %d", (long long)m, k);
    if (ldo < k) return fail(RTK_EINVAL, "ldo (%lld) < k (%d)", (long long)ldo, k);
    if (ldo >= (1LL << 30)) return fail(RTK_EINVAL, "ldo must be < 2^30, got %lld", (long long)ldo);
    if (dense && (ldd < m || ldd >= (1LL << 30)))
        return fail(RTK_EINVAL, "ldd must be in [m, 2^30), got %lld", (long long)ldd);
    if (idx8 && (ld8 < k || ld8 >= (1LL << 30))) return fail(RTK_EINVAL, "ld8 must be in [k, 2^30), got %lld", (long long)ld8);
    if (n > 0 && (!vals || !idx)) return fail(RTK_EINVAL, "vals/idx is NULL");
    if (!dense && !idx8) return fail(RTK_EINVAL, "dense and idx8 are both NULL (use rtk_rowtopk_*)");
    if (mode == rtk::kExact && hard_cap < 1) return fail(RTK_EINVAL, "hard_cap must be >= 1, got %d", hard_cap);
    if (mode == rtk::kEarly && max_iter < 1) return fail(RTK_EINVAL, "max_iter must be >= 1, got %d", max_iter);
    // native path: the paired-row kernel on unmasked tiles, vector loads and
    // stores (fp32 rows and dense rows 16-byte aligned; 16-bit rows 8-byte)
    // (each lane stores E = m / 32 contiguous dense elements: 16 bytes per
    // vector store, 8 for 16-bit rows of 128)
    const uintptr_t xa = dtype == 0 ? 16 : 8;
    const uintptr_t da = (dtype != 0 && m == 128) ? 8 : 16;
    const int64_t dq = (int64_t)da / (dtype == 0 ? 4 : 2);
    const bool ok = (m == 128 || m == 256) && k < m && n < 0xffff0000LL && ldx % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(x) % xa) == 0 &&
                    (!dense || (ldd % dq == 0 && (reinterpret_cast<uintptr_t>(dense) % da) == 0));
    if (!ok)
        return fail(RTK_EUNSUPPORTED, "shape outside the fused MaxK path (m=%lld, k=%d, ldx=%lld, ldd=%lld)",
                    (long long)m, k, (long long)ldx, (long long)ldd);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rc = reset_nan(nan_first_row, s);
    if (rc || n == 0) return rc;
    rtk::Args a = make_args(static_cast<const float*>(x), n, m, ldx, k, vals, idx, ldo, nullptr, nullptr,
                            nan_first_row);
    a.hard_cap = hard_cap;
    a.max_iter = max_iter;
    a.dense = dense;
    a.ldd = ldd;
    a.idx8 = idx8;
    a.ld8 = ld8;
    return rtk_dispatch_maxk(a, dtype, mode, s);
}

int rtk_exact_trace_f32(const float* x, int64_t n, int64_t m, int64_t ldx, int32_t k, double eps_rel,
                        int32_t hard_cap, int32_t* iters, int8_t* reasons, uint32_t* nan_first_row, void* stream) {
    return rowtopk_common(rtk::kTrace, x, n, m, ldx, k, eps_rel, hard_cap, 1, nullptr, nullptr, k, iters, reasons,
                          nan_first_row, stream);
}

int rtk_nan_scan_f32(const float* x, int64_t n, int64_t m, int64_t ldx, uint32_t* nan_first_row, void* stream) {
    int rc = check_common(x, n, m, ldx);
    if (rc) return rc;
    if (!nan_first_row) return fail(RTK_EINVAL, "nan_first_row is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rc = reset_nan(nan_first_row, s);
    if (rc || n == 0) return rc;
    rtk::Args a = make_args(x, n, m, ldx, 1, nullptr, nullptr, 1, nullptr, nullptr, nan_first_row);
    return launch_flat(rtk::nan_scan_kernel, a, s);
}

int rtk_row_min_max_f32(const float* x, int64_t n, int64_t m, int64_t ldx, float* mins, float* maxs, void* stream) {
    int rc = check_common(x, n, m, ldx);
    if (rc) return rc;
    if (n > 0 && (!mins || !maxs)) return fail(RTK_EINVAL, "mins/maxs is NULL");
    if (n == 0) return RTK_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rtk::Args a = make_args(x, n, m, ldx, 1, nullptr, nullptr, 1, nullptr, nullptr, nullptr);
    long long grid = (n + 7) / 8, cap = (long long)device_sms() * 8;
    if (grid > cap) grid = cap;
    rtk::min_max_kernel<<<(unsigned)grid, kFlatThreads, 0, s>>>(a, mins, maxs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

int rtk_count_ge_f32(const float* x, int64_t n, int64_t m, int64_t ldx, const float* thres, int32_t* counts,
                     void* stream) {
    int rc = check_common(x, n, m, ldx);
    if (rc) return rc;
    if (n > 0 && (!thres || !counts)) return fail(RTK_EINVAL, "thres/counts is NULL");
    if (n == 0) return RTK_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rtk::Args a = make_args(x, n, m, ldx, 1, nullptr, nullptr, 1, nullptr, nullptr, nullptr);
    long long grid = (n + 7) / 8, cap = (long long)device_sms() * 8;
    if (grid > cap) grid = cap;
    rtk::count_ge_kernel<<<(unsigned)grid, kFlatThreads, 0, s>>>(a, thres, counts);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

const char* rtk_last_error(void) { return g_err; }

int rtk_version(void) { return 100; }

int rtk_launch_shape(int64_t m, int32_t k, int32_t mode, int32_t* warps_per_cta, int32_t* ctas_per_sm_out,
                     int32_t* rows_per_warp) {
    if (m < 1 || m > 0x7fffffff || k < 1 || k > m || mode < 0 || mode > 2)
        return fail(RTK_EINVAL, "bad launch-shape query");
    // a 2^20-row, C-contiguous, 256-byte aligned matrix without traces (modes 0/1)
    alignas(256) static const float kDummy[64] = {};
    rtk::Args a = make_args(kDummy, 1 << 20, m, m, k, mode == rtk::kTrace ? nullptr : reinterpret_cast<float*>(256),
                            mode == rtk::kTrace ? nullptr : reinterpret_cast<int32_t*>(256), k,
                            mode == rtk::kTrace ? reinterpret_cast<int32_t*>(256) : nullptr,
                            mode == rtk::kTrace ? reinterpret_cast<int8_t*>(256) : nullptr, nullptr);
    int shape[3] = {0, 0, 0};
    int rc = RTK_OK;
    if (k == m) {
        shape[0] = kFlatThreads / 32;  // elementwise copy (_kernels.py:173-179)
    } else {
        rc = mode == rtk::kExact ? rtk_describe_exact(a, shape)
                                 : (mode == rtk::kEarly ? rtk_describe_early(a, shape) : rtk_describe_trace(a, shape));
    }
    if (warps_per_cta) *warps_per_cta = shape[0];
    if (ctas_per_sm_out) *ctas_per_sm_out = shape[1];
    if (rows_per_warp) *rows_per_warp = shape[2];
    return rc;
}

}  // extern "C"
