// rtk_dispatch_maxk.cu -- fused MaxK rows (rtk_maxk_dense): the paired-row
// kernel with DENSE = true, for M = 128 / 256 (E = 4 / 8, unmasked tiles),
// fp32 or 16-bit rows; rtk_maxk_dense checks the shape (include/rtk.h).
#include "rtk_dispatch.cuh"

namespace {

template <int MODE, int E, class In>
int launch_maxk(const rtk::Args& a, cudaStream_t s) {
    using namespace rtk_dispatch;
    const size_t smem = (size_t)(kThreads / 32) * rtk::PairStage<E, true>::kWarpBytes;
    // one 256-bit (fp32) / 128-bit (16-bit) load per lane: E = 8 rows aligned to it
    const size_t align = std::is_same<In, float>::value ? 32 : 16;
    const bool wide = E == 8 && (reinterpret_cast<uintptr_t>(a.x) % align) == 0 && a.ldx % 8 == 0;
    if (wide) return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, false, true, In, true>, a, s, smem, kThreads, 2);
    return launch_rows(rtk::rowtopk_pair_kernel<MODE, E, false, false, In, true>, a, s, smem, kThreads, 2);
}

template <int MODE, class In>
int dispatch_maxk(const rtk::Args& a, cudaStream_t s) {
    return a.m == 128 ? launch_maxk<MODE, 4, In>(a, s) : launch_maxk<MODE, 8, In>(a, s);
}

template <class In>
int dispatch_mode(const rtk::Args& a, int mode, cudaStream_t s) {
    return mode == rtk::kExact ? dispatch_maxk<rtk::kExact, In>(a, s) : dispatch_maxk<rtk::kEarly, In>(a, s);
}

}  // namespace

int rtk_dispatch_maxk(const rtk::Args& a, int dtype, int mode, cudaStream_t s) {
    if (dtype == 0) return dispatch_mode<float>(a, mode, s);
    if (dtype == 1) return dispatch_mode<__nv_bfloat16>(a, mode, s);
    return dispatch_mode<__half>(a, mode, s);
}
