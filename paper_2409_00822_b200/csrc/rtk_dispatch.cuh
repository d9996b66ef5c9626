// rtk_dispatch.cuh -- kernel selection and launch for one mode (included by
// the per-mode translation units rtk_dispatch_{exact,early,trace}.cu, which
// nvcc compiles in parallel).  Chooses the tile / kernel for (M, alignment,
// traces), sizes the persistent grid from the occupancy of that
// instantiation and launches on the caller's stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rtk.h"
#include "rtk_big.cuh"
#include "rtk_kernels.cuh"
#include "rtk_pair.cuh"
#include "rtk_block.cuh"

// library-internal (rtk_capi.cu)
int rtk_fail(int code, const char* fmt, ...);
int rtk_device_sms();
int rtk_ctas_per_sm(const void* kernel, size_t smem, int threads);
int rtk_dispatch_exact(const rtk::Args& a, cudaStream_t s);
int rtk_dispatch_early(const rtk::Args& a, cudaStream_t s);
int rtk_dispatch_trace(const rtk::Args& a, cudaStream_t s);
int rtk_dispatch_x16(const rtk::Args& a, int dtype, int mode, cudaStream_t s);
int rtk_dispatch_maxk(const rtk::Args& a, int dtype, int mode, cudaStream_t s);
int rtk_describe_exact(const rtk::Args& a, int* shape3);
int rtk_describe_early(const rtk::Args& a, int* shape3);
int rtk_describe_trace(const rtk::Args& a, int* shape3);
bool rtk_encode_row_map(CUtensorMap* map, const float* x, long long n, int e, long long ldx);
bool rtk_encode_row_parts(CUtensorMap* maps, const float* x, long long n, int e, long long ldx, const int* widths,
                          int parts);

namespace rtk_dispatch {

template <class... T>
int fail(int code, const char* fmt, T... args) {
    return rtk_fail(code, fmt, args...);
}

#ifndef RTK_BIG_MIN_E
#define RTK_BIG_MIN_E 12  // smallest elements-per-lane tile routed to the long-row kernel
#endif
#ifndef RTK_PAIR_MAX_E
#define RTK_PAIR_MAX_E 8  // largest elements-per-lane tile routed to the paired-row kernel
#endif
constexpr int kThreads = RTK_CTA_THREADS;  // threads per CTA of the row kernels
constexpr int kFlatThreads = 256;         // threads per CTA of the elementwise kernels
constexpr size_t kMaxSmem = 227 * 1024;   // dynamic shared memory per CTA (sm_100 opt-in limit)


// Dry-run description of a launch (rtk_launch_shape): when set, the launch
// helpers record the chosen configuration here instead of launching.
struct LaunchShape {
    int warps_per_cta, ctas_per_sm, rows_per_warp;
};
inline thread_local LaunchShape* g_describe = nullptr;

inline bool describe(const void* kernel, size_t smem, int threads, int rows_per_warp) {
    if (!g_describe) return false;
    g_describe->warps_per_cta = threads / 32;
    g_describe->ctas_per_sm = rtk_ctas_per_sm(kernel, smem, threads);
    g_describe->rows_per_warp = rows_per_warp;
    return true;
}

template <class K>
int launch_rows(K kernel, const rtk::Args& a, cudaStream_t s, size_t smem, int threads = kThreads,
                int rows_per_warp = 1) {
    if (describe(reinterpret_cast<const void*>(kernel), smem, threads, rows_per_warp)) return RTK_OK;
    const long long warps_needed = a.n;
    const long long blocks_needed = (warps_needed + (threads / 32) - 1) / (threads / 32);
    long long grid = (long long)rtk_device_sms() * rtk_ctas_per_sm(reinterpret_cast<const void*>(kernel), smem, threads);
    if (grid > blocks_needed) grid = blocks_needed;
    if (grid < 1) grid = 1;
    kernel<<<(unsigned)grid, threads, smem, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

// Launch one row-kernel instantiation; traces are a template flag so the
// common no-trace launch carries no per-row trace stores.
template <int MODE, class Row>
int launch_row_kernel(const rtk::Args& a, cudaStream_t s, size_t smem) {
    if constexpr (MODE == rtk::kTrace) {
        return launch_rows(rtk::rowtopk_kernel<MODE, Row, true>, a, s, smem);
    } else {
        if ((a.iters != nullptr) != (a.reasons != nullptr))
            return fail(RTK_EINVAL, "iters and reasons must be both NULL or both non-NULL");
        if (a.iters != nullptr) return launch_rows(rtk::rowtopk_kernel<MODE, Row, true>, a, s, smem);
        return launch_rows(rtk::rowtopk_kernel<MODE, Row, false>, a, s, smem);
    }
}

template <int MODE, int V, int C>
int launch_reg(const rtk::Args& a, cudaStream_t s) {
    // staging buffer: k (value, index) pairs per warp (no selection in trace mode)
    const size_t smem = MODE == rtk::kTrace ? 0 : (size_t)(kThreads / 32) * rtk::RegRow<V, C, false>::stage_bytes(a.k);
    if (a.m == C * 32 * V) return launch_row_kernel<MODE, rtk::RegRow<V, C, false>>(a, s, smem);
    return launch_row_kernel<MODE, rtk::RegRow<V, C, true>>(a, s, smem);
}

// Long rows (rtk_big.cuh): one register tile, cp.async ring, k-pair staging.
template <int MODE, int E, bool MASKED, bool TRACES>
int launch_big_kernel(const rtk::Args& a, cudaStream_t s) {
    using Row = rtk::LaneRowCut<E, MASKED>;
    // warps per CTA: BigThreads, fewer when k pairs + ring of 8 warps would
    // not fit in shared memory (the kernel reads its warp count from blockDim)
    const size_t per_warp = Row::stage_bytes(a.k) + RTK_BIG_DEPTH * Row::kRowBytes;
    int wpc = rtk::BigThreads<E>::value / 32;
    while (wpc > 1 && (size_t)wpc * per_warp > kMaxSmem) --wpc;
    const int threads = 32 * wpc;
    const size_t smem = (size_t)wpc * per_warp;
    return launch_rows(rtk::rowtopk_big_kernel<MODE, E, MASKED, TRACES>, a, s, smem, threads);
}

// TMA staging for unmasked long rows with E = 16 / 32 (rtk_big.cuh).
#ifndef RTK_USE_TMA
#define RTK_USE_TMA 1
#endif
template <int MODE, int E, bool TRACES>
int launch_big_tma_kernel(const rtk::Args& a, cudaStream_t s, const CUtensorMap& map) {
    using Row = rtk::TmaRow<E>;
    constexpr int wpc = RTK_BIG_THREADS / 32;
    const size_t smem = (size_t)wpc * Row::stage_bytes(a.k) + Row::kSlotAlign + (size_t)wpc * (Row::kSlotBytes + 8);
    auto kernel = rtk::rowtopk_big_tma_kernel<MODE, E, TRACES>;
    if (describe(reinterpret_cast<const void*>(kernel), smem, RTK_BIG_THREADS, 1)) return RTK_OK;
    const long long blocks_needed = (a.n + wpc - 1) / wpc;
    long long grid = (long long)rtk_device_sms() * rtk_ctas_per_sm(reinterpret_cast<const void*>(kernel), smem,
                                                                   RTK_BIG_THREADS);
    if (grid > blocks_needed) grid = blocks_needed;
    if (grid < 1) grid = 1;
    kernel<<<(unsigned)grid, RTK_BIG_THREADS, smem, s>>>(a, map);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

// Paired long rows on TMA slots (rtk_big.cuh): E = 16, no traces, exact
// with eps_rel = 0 or early stop.
template <int MODE, int E, int CMAX = 4>
int launch_big_pair_tma_kernel(const rtk::Args& a, cudaStream_t s, const CUtensorMap& map, const CUtensorMap& map1,
                               const CUtensorMap& map2) {
    if constexpr (CMAX == 4 && MODE == rtk::kExact && E >= RTK_CAND8_MIN_E) {  // the 8-slot candidate search, own kernel
        if (rtk::long_cand8<E>(a.k)) return launch_big_pair_tma_kernel<MODE, E, 8>(a, s, map, map1, map2);
    }
    using Row = rtk::TmaRow<E>;
    constexpr int wpc = RTK_BIG_THREADS / 32;
    const size_t smem =
        (size_t)wpc * 2 * rtk::pair_stage_bytes<Row>(a.k) + Row::kSlotAlign + (size_t)wpc * (2 * Row::kSlotBytes + 8);
    auto kernel = rtk::rowtopk_big_pair_tma_kernel<MODE, E, CMAX>;
    if (describe(reinterpret_cast<const void*>(kernel), smem, RTK_BIG_THREADS, 2)) return RTK_OK;
    const long long blocks_needed = (a.n + 2 * wpc - 1) / (2 * wpc);
    long long grid = (long long)rtk_device_sms() * rtk_ctas_per_sm(reinterpret_cast<const void*>(kernel), smem,
                                                                   RTK_BIG_THREADS);
    if (grid > blocks_needed) grid = blocks_needed;
    if (grid < 1) grid = 1;
    kernel<<<(unsigned)grid, RTK_BIG_THREADS, smem, s>>>(a, map, map1, map2);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

// Paired long rows through the cp.async ring (rtk_big.cuh): E <= 32 rows the
// TMA path does not take (E = 12..28, masked rows).
#ifndef RTK_BIG_PAIR_CP
#define RTK_BIG_PAIR_CP 1
#endif
template <int MODE, int E, bool MASKED, int CMAX = 4>
int launch_big_pair_kernel(const rtk::Args& a, cudaStream_t s) {
    if constexpr (CMAX == 4 && MODE == rtk::kExact && E >= RTK_CAND8_MIN_E) {  // the 8-slot candidate search
        if (rtk::long_cand8<E>(a.k)) return launch_big_pair_kernel<MODE, E, MASKED, 8>(a, s);
    }
    using Row = rtk::LaneRowCut<E, MASKED>;
    const size_t per_warp = 2 * (rtk::pair_stage_bytes<Row>(a.k) + Row::kRowBytes);
    constexpr int wpc = RTK_BIG_THREADS / 32;
    return launch_rows(rtk::rowtopk_big_pair_kernel<MODE, E, MASKED, float, CMAX>, a, s, (size_t)wpc * per_warp, RTK_BIG_THREADS, 2);
}

// Early stop with k >= 128 stays on the single-row kernel at E <= 16 (two
// k-pair flushes per step measured 5-6% slower paired there); from E = 20 up
// the paired kernel is faster (M = 768: -13%, M = 640 / 1024: -2..3%).
template <int MODE, int E>
bool big_pair_eligible(const rtk::Args& a) {
    return MODE != rtk::kTrace && a.iters == nullptr && a.reasons == nullptr && a.n < (1LL << 30) &&
           (MODE == rtk::kEarly ? (a.k < 128 || E > 16) : a.eps_rel == 0.0);
}

#ifndef RTK_TMA_SPLIT
#define RTK_TMA_SPLIT 1
#endif
template <int MODE, int E, bool MASKED>
int launch_big(const rtk::Args& a, cudaStream_t s) {
    if constexpr (RTK_USE_TMA && RTK_BIG_PAIR && RTK_TMA_SPLIT && !MASKED && rtk::TmaParts<E>::kSplit &&
                  MODE != rtk::kTrace) {
        // paired rows only: one tensor copy per 16 / 8 / 4-float part of each lane row (TmaRow)
        using P = rtk::TmaParts<E>;
        const int widths[3] = {P::w0, P::w1, P::w2};
        CUtensorMap m[3];
        if (big_pair_eligible<MODE, E>(a) && a.n < (1LL << 31) && rtk_encode_row_parts(m, a.x, a.n, E, a.ldx, widths, P::n))
            return launch_big_pair_tma_kernel<MODE, E>(a, s, m[0], P::n > 1 ? m[1] : m[0], P::n > 2 ? m[2] : m[0]);
    }
    if constexpr (RTK_USE_TMA && !MASKED && (E == 16 || E == 32)) {
        CUtensorMap map;
        if (a.n < (1LL << 31) && rtk_encode_row_map(&map, a.x, a.n, E, a.ldx)) {
#ifndef RTK_BIG_PAIR_E32
#define RTK_BIG_PAIR_E32 1
#endif
            if constexpr (RTK_BIG_PAIR && (E == 16 || (RTK_BIG_PAIR_E32 && E == 32)) && MODE != rtk::kTrace) {
                if (big_pair_eligible<MODE, E>(a)) return launch_big_pair_tma_kernel<MODE, E>(a, s, map, map, map);
            }
            if constexpr (MODE == rtk::kTrace) {
                return launch_big_tma_kernel<MODE, E, true>(a, s, map);
            } else {
                if ((a.iters != nullptr) != (a.reasons != nullptr))
                    return fail(RTK_EINVAL, "iters and reasons must be both NULL or both non-NULL");
                if (a.iters != nullptr) return launch_big_tma_kernel<MODE, E, true>(a, s, map);
                return launch_big_tma_kernel<MODE, E, false>(a, s, map);
            }
        }
    }
    if constexpr (RTK_BIG_PAIR_CP && E <= 32 && MODE != rtk::kTrace) {
        if (big_pair_eligible<MODE, E>(a)) return launch_big_pair_kernel<MODE, E, MASKED>(a, s);
    }
    if constexpr (MODE == rtk::kTrace) {
        return launch_big_kernel<MODE, E, MASKED, true>(a, s);
    } else {
        if ((a.iters != nullptr) != (a.reasons != nullptr))
            return fail(RTK_EINVAL, "iters and reasons must be both NULL or both non-NULL");
        if (a.iters != nullptr) return launch_big_kernel<MODE, E, MASKED, true>(a, s);
        return launch_big_kernel<MODE, E, MASKED, false>(a, s);
    }
}

// Paired-row kernel (rtk_pair.cuh): launches without traces; exact mode
// only with eps_rel == 0.
template <int MODE, int E>
bool pair_eligible(const rtk::Args& a) {
    if constexpr (MODE == rtk::kTrace || E > RTK_PAIR_MAX_E) {
        return false;
    } else {
        if (a.iters != nullptr || a.reasons != nullptr) return false;
        if (a.n >= 0xffff0000LL) return false;  // 32-bit row cursors: n + 2 * (warps in the grid) < 2^32
        return MODE == rtk::kEarly || a.eps_rel == 0.0;
    }
}

template <int MODE, int E>
int launch_pair(const rtk::Args& a, cudaStream_t s) {
    if constexpr (MODE == rtk::kTrace || E > RTK_PAIR_MAX_E) {
        return fail(RTK_EINVAL, "internal: paired-row kernel not instantiated");
    } else {
        // two selection staging buffers per warp
        const size_t smem = (size_t)(kThreads / 32) * 2 * rtk::LaneRow<E, false>::kStageBytes;
        const bool wide = (reinterpret_cast<uintptr_t>(a.x) & 31) == 0 && a.ldx % 8 == 0;  // 256-bit loads
        if (a.m == 32 * E && wide)
            return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, false, true>, a, s, smem, kThreads, 2);
        if (a.m == 32 * E) return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, false, false>, a, s, smem, kThreads, 2);
        return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, true, false>, a, s, smem, kThreads, 2);
    }
}

template <int MODE, int E>
int launch_lane(const rtk::Args& a, cudaStream_t s) {
    if (pair_eligible<MODE, E>(a)) return launch_pair<MODE, E>(a, s);
    // Long rows: one register tile fed by a shared-memory ring (rtk_big.cuh).
    if constexpr (E >= RTK_BIG_MIN_E) {
        if (a.m == 32 * E) return launch_big<MODE, E, false>(a, s);
        return launch_big<MODE, E, true>(a, s);
    } else {
        // staging buffer per warp: row copy + 32*E indices (no selection in trace mode)
        const size_t smem = MODE == rtk::kTrace ? 0 : (size_t)(kThreads / 32) * rtk::LaneRow<E, false>::kStageBytes;
        const bool wide = (reinterpret_cast<uintptr_t>(a.x) & 31) == 0 && a.ldx % 8 == 0;  // 256-bit loads
        if (a.m == 32 * E && wide) return launch_row_kernel<MODE, rtk::LaneRow<E, false, true>>(a, s, smem);
        if (a.m == 32 * E) return launch_row_kernel<MODE, rtk::LaneRow<E, false, false>>(a, s, smem);
        return launch_row_kernel<MODE, rtk::LaneRow<E, true, false>>(a, s, smem);
    }
}

// Longest rows (rtk_block.cuh): one CTA of W warps per row, 4096 < M <= 8192;
// each lane holds E = CAP / (32 W) elements (CAP = 6144 or 8192 columns).
// W = 2 measured best in exact mode, W = 4 with early stop.
#ifdef RTK_BLOCK_W
template <int MODE>
constexpr int kBlockW = RTK_BLOCK_W;
#else
template <int MODE>
constexpr int kBlockW = MODE == rtk::kEarly ? 4 : 2;
#endif
template <int MODE, int W, int E, bool TRACES>
int launch_block_kernel(const rtk::Args& a, cudaStream_t s) {
    using Tile = rtk::LaneRow<E, true, false>;
    const int threads = W * 32;
    const size_t smem = (((size_t)8 * a.k + 15) & ~(size_t)15) + (size_t)W * Tile::kRowBytes;
    auto kernel = rtk::rowtopk_block_kernel<MODE, W, E, TRACES>;
    if (describe(reinterpret_cast<const void*>(kernel), smem, threads, 0)) return RTK_OK;  // W warps per row
    long long grid = (long long)rtk_device_sms() * rtk_ctas_per_sm(reinterpret_cast<const void*>(kernel), smem, threads);
    if (grid > a.n) grid = a.n;
    if (grid < 1) grid = 1;
    kernel<<<(unsigned)grid, threads, smem, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RTK_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return RTK_OK;
}

template <int MODE, int W, int E>
int launch_block_e(const rtk::Args& a, cudaStream_t s) {
    if constexpr (MODE == rtk::kTrace) {
        return launch_block_kernel<MODE, W, E, true>(a, s);
    } else {
        if ((a.iters != nullptr) != (a.reasons != nullptr))
            return fail(RTK_EINVAL, "iters and reasons must be both NULL or both non-NULL");
        if (a.iters != nullptr) return launch_block_kernel<MODE, W, E, true>(a, s);
        return launch_block_kernel<MODE, W, E, false>(a, s);
    }
}

template <int MODE, int W>
int launch_block(const rtk::Args& a, cudaStream_t s) {
    if (a.m <= 6144) return launch_block_e<MODE, W, 6144 / (32 * W)>(a, s);
    return launch_block_e<MODE, W, 8192 / (32 * W)>(a, s);
}

template <int MODE>
int dispatch(const rtk::Args& a, cudaStream_t s) {
    const int m = a.m;
    const bool vec4 = (m % 4 == 0) && (a.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
#ifdef RTK_TUNE_BLOCK  // tuning builds: only the CTA-per-row kernel (M > 4096)
    if (m > 4096 && m <= 8192 && vec4) return launch_block<MODE, kBlockW<MODE>>(a, s);
    return launch_row_kernel<MODE, rtk::GlobalRow>(a, s, 0);
#elif defined(RTK_TUNE_E)  // tuning builds: only one register-tile width (fast to compile)
    if (m <= 1024 && vec4 && (m + 127) / 128 * 4 == RTK_TUNE_E) return launch_lane<MODE, RTK_TUNE_E>(a, s);
    return launch_row_kernel<MODE, rtk::GlobalRow>(a, s, 0);
#else
    if (m <= 1024 && vec4) {
        // elements per lane: ceil(m / 32) rounded up to a multiple of 4
        switch ((m + 127) / 128) {
            case 1: return launch_lane<MODE, 4>(a, s);
            case 2: return launch_lane<MODE, 8>(a, s);
            case 3: return launch_lane<MODE, 12>(a, s);
            case 4: return launch_lane<MODE, 16>(a, s);
            case 5: return launch_lane<MODE, 20>(a, s);
            case 6: return launch_lane<MODE, 24>(a, s);
            case 7: return launch_lane<MODE, 28>(a, s);
            default: return launch_lane<MODE, 32>(a, s);
        }
    }
    if (m <= 1024) {
        const int c = (m + 31) / 32;
        if (c <= 1) return launch_reg<MODE, 1, 1>(a, s);
        if (c <= 2) return launch_reg<MODE, 1, 2>(a, s);
        if (c <= 4) return launch_reg<MODE, 1, 4>(a, s);
        if (c <= 8) return launch_reg<MODE, 1, 8>(a, s);
        if (c <= 16) return launch_reg<MODE, 1, 16>(a, s);
        return launch_reg<MODE, 1, 32>(a, s);
    }
    if (m <= 4096 && vec4) {
        // still one warp per row: E = 48 / 64 / 96 / 128 elements per lane
        if (m <= 1536) return launch_lane<MODE, 48>(a, s);
        if (m <= 2048) return launch_lane<MODE, 64>(a, s);
        if (m <= 3072) return launch_lane<MODE, 96>(a, s);
        return launch_lane<MODE, 128>(a, s);
    }
    if (m <= 8192 && vec4) return launch_block<MODE, kBlockW<MODE>>(a, s);  // CTA per row
    return launch_row_kernel<MODE, rtk::GlobalRow>(a, s, 0);
#endif
}


// The configuration dispatch<MODE> would launch for `a` (no launch).
template <int MODE>
int describe_dispatch(const rtk::Args& a, int* shape3) {
    LaunchShape sh{0, 0, 0};
    g_describe = &sh;
    const int rc = dispatch<MODE>(a, nullptr);
    g_describe = nullptr;
    shape3[0] = sh.warps_per_cta;
    shape3[1] = sh.ctas_per_sm;
    shape3[2] = sh.rows_per_warp;
    return rc;
}

}  // namespace rtk_dispatch
