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
#include "rtk_pair.cuh"

namespace rtk {

#ifndef RTK_BIG_DEPTH
#define RTK_BIG_DEPTH 1  // row buffers per warp in the cp.async ring
#endif
#ifndef RTK_BIG_THREADS
#define RTK_BIG_THREADS 256
#endif

// Threads per CTA and minimum resident CTAs per SM requested from ptxas.
// E <= 32 (256 threads): caps registers at ~64 (E = 24..32; ~85 with
// masking), ~51 (E = 16..20), ~42 (E = 12).  Rows past 1024 columns keep
// one warp per row with E = 48..128 elements per lane (128 threads): the cap
// is about E + 64 registers (16 resident warps at E <= 64, 12 at 96, 8 at 128).
#ifndef RTK_BIG_WIDE_THREADS
#define RTK_BIG_WIDE_THREADS 256  // CTA size for E > 32
#endif
template <int E>
struct BigThreads {
    static constexpr int value = E > 32 ? RTK_BIG_WIDE_THREADS : RTK_BIG_THREADS;
};
template <int E, bool MASKED>
struct BigMinCtas {
    static constexpr int wide = 65536 / (BigThreads<E>::value * (E + 64));
    static constexpr int value = E <= 12 ? 6 : (E <= 20 ? 5 : (E <= 32 ? (MASKED ? 3 : 4) : (wide > 0 ? wide : 1)));
};

// In: the input element type (float, or __nv_bfloat16 / __half for
// rtk_rowtopk_x16: 16-bit chunks in the ring, widened when the tile is read).
template <int MODE, int E, bool MASKED, bool TRACES, class In = float>
__global__ void __launch_bounds__(BigThreads<E>::value, BigMinCtas<E, MASKED>::value) rowtopk_big_kernel(Args a) {
    using Row = LaneRowCut<E, MASKED>;
    constexpr bool kF32 = std::is_same<In, float>::value;
    constexpr unsigned kSlot = kF32 ? Row::kRowBytes : Row::kRowBytes16;
    const In* __restrict__ x = reinterpret_cast<const In*>(a.x);
    constexpr int D = RTK_BIG_DEPTH;
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned wpc = blockDim.x >> 5;
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned stage_bytes = Row::stage_bytes(a.k);  // k (value, index) pairs
    const unsigned sbase = base + (unsigned)wid * stage_bytes;
    const unsigned ring = base + wpc * stage_bytes + (unsigned)wid * D * kSlot;
    const unsigned nw = gridDim.x * wpc;
    const unsigned long long n = (unsigned long long)a.n;
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const unsigned ldx_b = (unsigned)a.ldx * (unsigned)sizeof(In);
    const bool fp = a.eps_rel == 0.0;
    if constexpr (MASKED) {  // padding chunks of the ring: NaN once (load_smem_prefilled)
#pragma unroll
        for (int d = 0; d < D; ++d) Row::fill_slot_nan(ring + d * kSlot, lane, kSlot);
        __syncwarp();
    }
    auto stage = [&](unsigned row, unsigned slot, unsigned salt) {
        if constexpr (kF32)
            Row::stage_async(row_ptr(x, row, ldx_b), a.m, lane, slot, salt);
        else
            Row::template stage_async16<In>(row_ptr(x, row, ldx_b), a.m, lane, slot, salt);
    };
    // prologue: rows r, r + nw, ..., r + (D-1) nw
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const unsigned long long rd = (unsigned long long)r + (unsigned long long)d * nw;
        if (rd < n) stage((unsigned)rd, ring + d * kSlot, 0u);
        cp_async_commit();
    }
    unsigned slot = 0;
    Row row;
    for (;;) {
        cp_async_wait<D - 1>();  // this lane's copies of this row have landed ...
        __syncwarp();            // ... and (chunks go to their owner lanes) every lane's
        const unsigned sl = ring + slot * kSlot;
        if constexpr (kF32)
            row.load_smem_prefilled(sl, lane);
        else
            row.template load_smem16<In>(sl, lane);
        const unsigned long long rpre = (unsigned long long)r + (unsigned long long)D * nw;
        // refill after the tile has been read (the token orders the LDGSTS after the LDS)
        process_row<MODE, TRACES>(row, r, a, lane, sbase, fp, [&](unsigned tok) {
            __syncwarp();  // every lane has read its tile out of the slot before any refill lands
            const unsigned salt = tok & a.opaque_zero;
            if (rpre < n) stage((unsigned)rpre + salt, sl, salt);
            cp_async_commit();
        });
        if ((unsigned long long)r + nw >= n) break;
        r += nw;
        slot = slot + 1 == D ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

// Paired long rows through the cp.async ring (E = 12..32 incl. masked rows,
// where the TMA map does not apply): two ring slots per warp, refilled with
// the next pair once both tiles are in registers; same pair scheme as above.
// fp32 E <= 16: 4 CTAs (64 registers), except exact mode at E = 16, where 3
// (80 registers, no candidate-search spills) measured 3% faster (and 2-3%
// slower at E = 12).  16-bit rows need the widening registers too: 128.
template <int MODE, int E, class In>
struct BigPairCpMinCtas {
    static constexpr int value = (E <= 16 && std::is_same<In, float>::value) ? (MODE == kExact && E == 16 ? 3 : 4) : 2;
};

template <int MODE, int E, bool MASKED, class In = float, int CMAX = 4>
__global__ void __launch_bounds__(RTK_BIG_THREADS, BigPairCpMinCtas<MODE, E, In>::value) rowtopk_big_pair_kernel(Args a) {
    using Row = LaneRowCut<E, MASKED>;
    constexpr bool kF32 = std::is_same<In, float>::value;
    constexpr unsigned kSlot = kF32 ? Row::kRowBytes : Row::kRowBytes16;
    const In* __restrict__ x = reinterpret_cast<const In*>(a.x);
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned wpc = blockDim.x >> 5;
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned stage_bytes = pair_stage_bytes<Row>(a.k);  // k-pair staging or the candidate set
    const unsigned sA = base + (unsigned)wid * 2u * stage_bytes;
    const unsigned sB = sA + stage_bytes;
    const unsigned ringA = base + wpc * 2u * stage_bytes + (unsigned)wid * 2u * kSlot;
    const unsigned ringB = ringA + kSlot;
    const unsigned nw = gridDim.x * wpc;
    const unsigned n = (unsigned)a.n;  // the host guarantees n + 2 nw < 2^31
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const unsigned last = n - 1;
    const unsigned ldx_b = (unsigned)a.ldx * (unsigned)sizeof(In);
    const int steps = MODE == kEarly ? a.max_iter : min(a.hard_cap, RTK_FAST_STEPS);
    if constexpr (MASKED) {  // padding chunks: NaN once (load_smem_prefilled / NaN halves)
        Row::fill_slot_nan(ringA, lane, kSlot);
        Row::fill_slot_nan(ringB, lane, kSlot);
        __syncwarp();
    }
    auto stage = [&](unsigned row, unsigned slot, unsigned salt) {
        if constexpr (kF32)
            Row::stage_async(row_ptr(x, row, ldx_b), a.m, lane, slot, salt);
        else
            Row::template stage_async16<In>(row_ptr(x, row, ldx_b), a.m, lane, slot, salt);
    };
    auto load = [&](Row& R, unsigned slot) {
        if constexpr (kF32)
            R.load_smem_prefilled(slot, lane);
        else
            R.template load_smem16<In>(slot, lane);
    };
    stage(r, ringA, 0u);
    stage(min(r + nw, last), ringB, 0u);
    cp_async_commit();
    Row A, B;
    for (;;) {
        cp_async_wait<0>();  // this lane's copies have landed ...
        __syncwarp();        // ... and every lane's (chunks go to their owner lanes)
        load(A, ringA);
        load(B, ringB);
        const unsigned rn = r + 2u * nw;
        process_pair<MODE, false, In, CMAX>(A, B, r, r + nw, r + nw < n, a, lane, sA, sB, steps, [&](unsigned tok) {
            __syncwarp();  // every lane has read both slots before any refill lands
            const unsigned salt = tok & a.opaque_zero;
            if (rn < n) {
                stage(rn + salt, ringA, salt);
                stage(min(rn + nw, last) + salt, ringB, salt);
            }
            cp_async_commit();
        });
        if (rn >= n) break;
        r = rn;
    }
    cp_async_wait<0>();
}

}  // namespace rtk

// ---------------------------------------------------------------------------
// TMA variant (unmasked rows, E = 16 or 32): one elected lane per warp loads
// the whole next row into the warp's slot with a tensor-map bulk copy
// (cp.async.bulk.tensor, completion on an mbarrier), the tensor map views the
// matrix as [n][32][E] floats and applies the hardware swizzle that makes the
// lane-contiguous LDS.128 reads conflict-free without padding (128B swizzle:
// 16-byte chunk c of lane l sits at c ^ (l & 7); 64B: c ^ ((l >> 1) & 3)).
#include <cuda.h>

namespace rtk {

// Split widths (paired kernel only): lane rows of 48-112 bytes fit no
// swizzle, so each row arrives as up to three tensor copies of 16 / 8 / 4
// floats per lane -- 16 with 64B swizzle, 8 with 32B swizzle (chunk c of
// lane l at c ^ ((l >> 2) & 1)), 4 unswizzled -- into consecutive parts of
// the slot.
template <int E>
struct TmaParts {
    // E = 24 only: the 4-float parts of E = 12 / 20 / 28 (16-byte boxes)
    // measured 4-7% slower in exact mode and 26-33% slower in early stop than
    // the cp.async ring
    static constexpr bool kSplit = E == 24;
    static constexpr int w0 = kSplit ? (E >= 16 ? 16 : 8) : E;
    static constexpr int w1 = kSplit ? (E >= 16 ? ((E - 16) >= 8 ? 8 : E - 16) : E - 8) : 0;
    static constexpr int w2 = kSplit ? E - w0 - w1 : 0;
    static constexpr int n = 1 + (w1 > 0) + (w2 > 0);
    __host__ __device__ static constexpr int width(int i) { return i == 0 ? w0 : (i == 1 ? w1 : w2); }
    __host__ __device__ static constexpr int first(int i) { return i == 0 ? 0 : (i == 1 ? w0 : w0 + w1); }
    static_assert(!kSplit || ((w1 == 0 || w1 == 8 || w1 == 4) && (w2 == 0 || w2 == 4)), "split TMA rows: 16 / 8 / 4 parts");
};

template <int E>
struct TmaRow : LaneRowCut<E, false> {
    using Parts = TmaParts<E>;
    static constexpr unsigned kSlotBytes = 32u * E * 4u;   // raw row, swizzled in place
    static constexpr unsigned kSlotAlign = E == 32 ? 1024u : 512u;
    __device__ __forceinline__ static unsigned phys_chunk(int l, int c) {
        return E == 32 ? (unsigned)(c ^ (l & 7)) : (unsigned)(c ^ ((l >> 1) & 3));
    }
    template <int W>
    __device__ __forceinline__ static unsigned part_chunk(int l, int c) {
        return W == 16 ? (unsigned)(c ^ ((l >> 1) & 3)) : (W == 8 ? (unsigned)(c ^ ((l >> 2) & 1)) : (unsigned)c);
    }
    template <int P>
    __device__ __forceinline__ void load_part(unsigned slot, int lane) {
        constexpr int W = Parts::width(P), Q = Parts::first(P);
        if constexpr (W > 0) {
            const unsigned b = slot + 32u * 4u * (unsigned)Q + (unsigned)lane * 4u * W;
#pragma unroll
            for (int c = 0; c < W / 4; ++c) {
                const float4 q = lds128(b + 16u * part_chunk<W>(lane, c));
                this->v[Q + 4 * c] = q.x;
                this->v[Q + 4 * c + 1] = q.y;
                this->v[Q + 4 * c + 2] = q.z;
                this->v[Q + 4 * c + 3] = q.w;
            }
        }
    }
    __device__ __forceinline__ void load_swizzled(unsigned slot, int lane) {
        if constexpr (Parts::kSplit) {
            load_part<0>(slot, lane);
            load_part<1>(slot, lane);
            load_part<2>(slot, lane);
            return;
        }
        const unsigned base = slot + (unsigned)lane * E * 4u;
#pragma unroll
        for (int c = 0; c < E / 4; ++c) {
            const float4 q = lds128(base + 16u * phys_chunk(lane, c));
            this->v[4 * c] = q.x;
            this->v[4 * c + 1] = q.y;
            this->v[4 * c + 2] = q.z;
            this->v[4 * c + 3] = q.w;
        }
    }
};

__device__ __forceinline__ void mbar_init(unsigned bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_row(unsigned slot, const CUtensorMap* map, int row, unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(slot),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(0), "r"(0), "r"(row), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                     : "=r"(done)
                     : "r"(bar), "r"(phase)
                     : "memory");
    } while (!done);
}

template <int MODE, int E, bool TRACES>
__global__ void __launch_bounds__(RTK_BIG_THREADS, BigMinCtas<E, false>::value)
    rowtopk_big_tma_kernel(Args a, const __grid_constant__ CUtensorMap map) {
    using Row = TmaRow<E>;
    extern __shared__ __align__(16) float smem[];  // slots are aligned by hand (kSlotAlign)
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned wpc = blockDim.x >> 5;
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned stage_bytes = Row::stage_bytes(a.k);
    const unsigned slots = (base + wpc * stage_bytes + Row::kSlotAlign - 1) & ~(Row::kSlotAlign - 1);
    const unsigned slot = slots + (unsigned)wid * Row::kSlotBytes;
    const unsigned bar = slots + wpc * Row::kSlotBytes + 8u * (unsigned)wid;
    const unsigned sbase = base + (unsigned)wid * stage_bytes;
    const unsigned nw = gridDim.x * wpc;
    const unsigned long long n = (unsigned long long)a.n;
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const bool fp = a.eps_rel == 0.0;
    if (lane == 0) {
        mbar_init(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_row(slot, &map, (int)r, bar, Row::kSlotBytes);
    }
    __syncwarp();
    unsigned phase = 0;
    Row row;
    for (;;) {
        mbar_wait(bar, phase);
        phase ^= 1u;
        row.load_swizzled(slot, lane);
        const unsigned long long rn = (unsigned long long)r + nw;
        process_row<MODE, TRACES>(row, r, a, lane, sbase, fp, [&](unsigned tok) {
            __syncwarp();  // every lane has read the slot
            if (lane == 0 && rn < n) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_row(slot, &map, (int)(rn + (tok & a.opaque_zero)), bar, Row::kSlotBytes);
            }
        });
        if (rn >= n) break;
        r = (unsigned)rn;
    }
}

// Paired long rows (E = 16 or 32: M = 512 / 1024, unmasked; exact with eps_rel = 0 or early stop,
// no traces): the row-pair scheme of rtk_pair.cuh (both rows' bisection steps
// interleaved, one FADD2 + FMUL2 for both midpoints, one f32x2 count tree)
// on tiles fed by TMA: each warp owns two swizzled row slots and one
// mbarrier; once both tiles are in registers (after the lane min/max) one
// elected lane issues the next pair's two tensor copies.
#ifndef RTK_BIG_PAIR
#define RTK_BIG_PAIR 1
#endif
__device__ __forceinline__ void tma_row_noarrive(unsigned slot, const CUtensorMap* map, int row, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(slot),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(0), "r"(0), "r"(row), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_pair(unsigned slotA, unsigned slotB, const CUtensorMap* map, int rowA, int rowB,
                                         unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2u * bytes) : "memory");
    tma_row_noarrive(slotA, map, rowA, bar);
    tma_row_noarrive(slotB, map, rowB, bar);
}
// both rows' slots of a pair: one tensor copy per row, or one per part
// (maps[0..2]) for the split widths
template <int E>
__device__ __forceinline__ void tma_pair_rows(unsigned slotA, unsigned slotB, const CUtensorMap* m0,
                                              const CUtensorMap* m1, const CUtensorMap* m2, int rowA, int rowB,
                                              unsigned bar) {
    using Parts = TmaParts<E>;
    tma_pair(slotA, slotB, m0, rowA, rowB, bar, TmaRow<E>::kSlotBytes);
    if constexpr (Parts::w1 > 0) {
        constexpr unsigned off = 32u * 4u * Parts::first(1);
        tma_row_noarrive(slotA + off, m1, rowA, bar);
        tma_row_noarrive(slotB + off, m1, rowB, bar);
    }
    if constexpr (Parts::w2 > 0) {
        constexpr unsigned off = 32u * 4u * Parts::first(2);
        tma_row_noarrive(slotA + off, m2, rowA, bar);
        tma_row_noarrive(slotB + off, m2, rowB, bar);
    }
}

// E = 16: 4 CTAs of 8 warps (64 registers) in early-stop mode, 3 (80
// registers) in exact mode, where the candidate-set search spilled at 64
// (measured 1.5-2.3% faster; early stop equal); E = 32: two 32-float tiles
// need ~100 registers.
template <int MODE, int E>
struct BigPairMinCtas {
    static constexpr int value = E == 16 ? (MODE == kExact ? 3 : 4) : (E < 16 ? 4 : 2);
};

template <int MODE, int E, int CMAX = 4>
__global__ void __launch_bounds__(RTK_BIG_THREADS, BigPairMinCtas<MODE, E>::value)
    rowtopk_big_pair_tma_kernel(Args a, const __grid_constant__ CUtensorMap map,
                                const __grid_constant__ CUtensorMap map1,  // split widths: parts 1 and 2
                                const __grid_constant__ CUtensorMap map2) {
    using Row = TmaRow<E>;
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned wpc = blockDim.x >> 5;
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned stage_bytes = pair_stage_bytes<Row>(a.k);  // k-pair staging or the candidate set
    const unsigned sA = base + (unsigned)wid * 2u * stage_bytes;
    const unsigned sB = sA + stage_bytes;
    const unsigned slots = (base + wpc * 2u * stage_bytes + Row::kSlotAlign - 1) & ~(Row::kSlotAlign - 1);
    const unsigned slotA = slots + (unsigned)wid * 2u * Row::kSlotBytes;
    const unsigned slotB = slotA + Row::kSlotBytes;
    const unsigned bar = slots + wpc * 2u * Row::kSlotBytes + 8u * (unsigned)wid;
    const unsigned nw = gridDim.x * wpc;
    const unsigned n = (unsigned)a.n;  // the host guarantees n + 2 nw < 2^31
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const unsigned last = n - 1;
    const int steps = MODE == kEarly ? a.max_iter : min(a.hard_cap, RTK_FAST_STEPS);
    if (lane == 0) {
        mbar_init(bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_pair_rows<E>(slotA, slotB, &map, &map1, &map2, (int)r, (int)min(r + nw, last), bar);
    }
    __syncwarp();
    unsigned phase = 0;
    Row A, B;
    for (;;) {
        mbar_wait(bar, phase);
        phase ^= 1u;
        A.load_swizzled(slotA, lane);
        B.load_swizzled(slotB, lane);
        const unsigned rn = r + 2u * nw;
        process_pair<MODE, false, float, CMAX>(A, B, r, r + nw, r + nw < n, a, lane, sA, sB, steps, [&](unsigned tok) {
            __syncwarp();  // every lane has read both slots
            if (lane == 0 && rn < n) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_pair_rows<E>(slotA, slotB, &map, &map1, &map2, (int)(rn + (tok & a.opaque_zero)),
                                 (int)min(rn + nw, last), bar);
            }
        });
        if (rn >= n) break;
        r = rn;
    }
}

}  // namespace rtk
