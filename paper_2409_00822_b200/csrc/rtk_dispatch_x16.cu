// rtk_dispatch_x16.cu -- 16-bit input rows (bfloat16 / float16), no traces
// (rtk_rowtopk_x16 checks the shape; see include/rtk.h): the paired-row
// kernel for M <= 256 (M % 4 == 0, 8-byte aligned rows) and the long-row
// kernel for 256 < M <= 4096 (M % 8 == 0, 16-byte aligned rows; 16-bit
// chunks in the cp.async ring, widened when the tile is read).
#include "rtk_dispatch.cuh"

namespace {

template <int MODE, int E, class In>
int launch_pair16(const rtk::Args& a, cudaStream_t s) {
    using namespace rtk_dispatch;
    const size_t smem = (size_t)(kThreads / 32) * 2 * rtk::LaneRow<E, false>::kStageBytes;
    // one 16-byte load per lane: E = 8, unmasked, 16-byte aligned rows
    const bool wide = E == 8 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && a.ldx % 8 == 0;
    if (a.m == 32 * E && wide)
        return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, false, true, In>, a, s, smem, kThreads, 2);
    if (a.m == 32 * E)
        return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, false, false, In>, a, s, smem, kThreads, 2);
    return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, true, false, In>, a, s, smem, kThreads, 2);
}

template <int MODE, int E, bool MASKED, class In>
int launch_big16_kernel(const rtk::Args& a, cudaStream_t s) {
    using namespace rtk_dispatch;
    using Row = rtk::LaneRowCut<E, MASKED>;
    const size_t per_warp = Row::stage_bytes(a.k) + RTK_BIG_DEPTH * Row::kRowBytes16;
    int wpc = rtk::BigThreads<E>::value / 32;
    while (wpc > 1 && (size_t)wpc * per_warp > kMaxSmem) --wpc;
    return launch_rows(rtk::rowtopk_big_kernel<MODE, E, MASKED, false, In>, a, s, (size_t)wpc * per_warp, 32 * wpc);
}

// Paired long rows (rtk_big.cuh, as rtk_dispatch.cuh's launch_big_pair_kernel)
template <int MODE, int E, bool MASKED, class In>
int launch_big16_pair_kernel(const rtk::Args& a, cudaStream_t s) {
    using namespace rtk_dispatch;
    using Row = rtk::LaneRowCut<E, MASKED>;
    const size_t per_warp = 2 * (rtk::pair_stage_bytes<Row>(a.k) + Row::kRowBytes16);
    constexpr int wpc = RTK_BIG_THREADS / 32;
    return launch_rows(rtk::rowtopk_big_pair_kernel<MODE, E, MASKED, In>, a, s, (size_t)wpc * per_warp,
                       RTK_BIG_THREADS, 2);
}

template <int MODE, int E, class In>
int launch_big16(const rtk::Args& a, cudaStream_t s) {
    // (paired 16-bit tiles spill above E = 20 even at 128 registers: E <= 20 only)
    if constexpr (RTK_BIG_PAIR_CP && E <= 20) {
        if (rtk_dispatch::big_pair_eligible<MODE, E>(a)) {
            if (a.m == 32 * E) return launch_big16_pair_kernel<MODE, E, false, In>(a, s);
            return launch_big16_pair_kernel<MODE, E, true, In>(a, s);
        }
    }
    if (a.m == 32 * E) return launch_big16_kernel<MODE, E, false, In>(a, s);
    return launch_big16_kernel<MODE, E, true, In>(a, s);
}

template <int MODE, class In>
int dispatch16(const rtk::Args& a, cudaStream_t s) {
    const int m = a.m;
    if (m <= 128) return launch_pair16<MODE, 4, In>(a, s);
    if (m <= 256) return launch_pair16<MODE, 8, In>(a, s);
    if (m <= 512) return launch_big16<MODE, 16, In>(a, s);
    if (m <= 768) return launch_big16<MODE, 24, In>(a, s);
    if (m <= 1024) return launch_big16<MODE, 32, In>(a, s);
    if (m <= 1536) return launch_big16<MODE, 48, In>(a, s);
    if (m <= 2048) return launch_big16<MODE, 64, In>(a, s);
    if (m <= 3072) return launch_big16<MODE, 96, In>(a, s);
    return launch_big16<MODE, 128, In>(a, s);
}

}  // namespace

int rtk_dispatch_x16(const rtk::Args& a, int dtype, int mode, cudaStream_t s) {
    if (dtype == 1)
        return mode == rtk::kExact ? dispatch16<rtk::kExact, __nv_bfloat16>(a, s)
                                   : dispatch16<rtk::kEarly, __nv_bfloat16>(a, s);
    return mode == rtk::kExact ? dispatch16<rtk::kExact, __half>(a, s) : dispatch16<rtk::kEarly, __half>(a, s);
}
