// rtk_big.cuh -- persistent row kernel for long rows (M > 256 on the
// lane-contiguous path, E >= 12 elements per lane).
//
// The register-double-buffered kernels hold two E-float tiles per lane; at
// E >= 12 that costs 66-123 registers and caps residency at 16-24 warps per
// SM.  Here a lane holds ONE tile: the next rows are staged in a per-warp
// ring of RTK_BIG_DEPTH row buffers in shared memory by cp.async (LDGSTS),
// refilled as soon as a row has been read into registers, and the
// selection stages only the first k (value, index) pairs (LaneRowCut), so
// both registers and shared memory stay small enough for 32-40 resident
// warps.  Same per-row path (process_row) and numeric contract as
// rowtopk_kernel; all modes, with or without traces.
#pragma once

#include "rtk_kernels.cuh"

namespace rtk {

#ifndef RTK_BIG_DEPTH
#define RTK_BIG_DEPTH 1  // row buffers per warp in the cp.async ring
#endif
#ifndef RTK_BIG_THREADS
#define RTK_BIG_THREADS 256
#endif

// Minimum resident CTAs (of RTK_BIG_THREADS) per SM requested from ptxas:
// caps registers at ~64 (E = 24..32; ~85 with masking), ~51 (E = 16..20), ~42 (E = 12).
template <int E, bool MASKED>
struct BigMinCtas {
    static constexpr int value = E <= 12 ? 6 : (E <= 20 ? 5 : (MASKED ? 3 : 4));
};

template <int MODE, int E, bool MASKED, bool TRACES>
__global__ void __launch_bounds__(RTK_BIG_THREADS, BigMinCtas<E, MASKED>::value) rowtopk_big_kernel(Args a) {
    using Row = LaneRowCut<E, MASKED>;
    constexpr int D = RTK_BIG_DEPTH;
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned wpc = blockDim.x >> 5;
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned stage_bytes = Row::stage_bytes(a.k);  // k (value, index) pairs
    const unsigned sbase = base + (unsigned)wid * stage_bytes;
    const unsigned ring = base + wpc * stage_bytes + (unsigned)wid * D * Row::kRowBytes;
    const unsigned nw = gridDim.x * wpc;
    const unsigned long long n = (unsigned long long)a.n;
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const unsigned ldx_b = (unsigned)a.ldx * 4u;
    const bool fp = a.eps_rel == 0.0;
    // prologue: rows r, r + nw, ..., r + (D-1) nw
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const unsigned long long rd = (unsigned long long)r + (unsigned long long)d * nw;
        if (rd < n) Row::stage_async(row_ptr(a.x, (unsigned)rd, ldx_b), a.m, lane, ring + d * Row::kRowBytes);
        cp_async_commit();
    }
    unsigned slot = 0;
    Row row;
    for (;;) {
        cp_async_wait<D - 1>();  // this lane's copies of this row have landed ...
        __syncwarp();            // ... and (chunks go to their owner lanes) every lane's
        const unsigned sl = ring + slot * Row::kRowBytes;
        row.load_smem(sl, a.m, lane);
        const unsigned long long rpre = (unsigned long long)r + (unsigned long long)D * nw;
        // refill after the tile has been read (the token orders the LDGSTS after the LDS)
        process_row<MODE, TRACES>(row, r, a, lane, sbase, fp, [&](unsigned tok) {
            __syncwarp();  // every lane has read its tile out of the slot before any refill lands
            if (rpre < n) Row::stage_async(row_ptr(a.x, (unsigned)rpre + (tok & a.opaque_zero), ldx_b), a.m, lane, sl);
            cp_async_commit();
        });
        if ((unsigned long long)r + nw >= n) break;
        r += nw;
        slot = slot + 1 == D ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

}  // namespace rtk
