// rtk_dispatch_x16.cu -- 16-bit input rows (bfloat16 / float16) on the
// paired-row kernel: M <= 256, M % 4 == 0, 8-byte aligned rows, no traces
// (rtk_rowtopk_x16 checks the shape; see include/rtk.h).
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

template <int MODE, class In>
int dispatch16(const rtk::Args& a, cudaStream_t s) {
    return a.m <= 128 ? launch_pair16<MODE, 4, In>(a, s) : launch_pair16<MODE, 8, In>(a, s);
}

}  // namespace

int rtk_dispatch_x16(const rtk::Args& a, int dtype, int mode, cudaStream_t s) {
    if (dtype == 1)
        return mode == rtk::kExact ? dispatch16<rtk::kExact, __nv_bfloat16>(a, s)
                                   : dispatch16<rtk::kEarly, __nv_bfloat16>(a, s);
    return mode == rtk::kExact ? dispatch16<rtk::kExact, __half>(a, s) : dispatch16<rtk::kEarly, __half>(a, s);
}
