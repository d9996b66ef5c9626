// rtk_block.cuh -- one CTA per row for the longest rows (4096 < M <= 8192 on
// the vectorised path; the reference's validated regime ends at 8192
// columns, batch.py:27).  Rows up to 4096 columns stay one warp per row
// (rtk_big.cuh with E up to 128 elements per lane), which measured faster:
// every reduction here costs a block barrier.
//
// W warps share a row: thread t of the CTA holds the E = 8192 / (32 W)
// consecutive elements [t E, (t+1) E) in registers (the LaneRow layout with
// the lane index taken over the whole CTA), so the per-step work of a warp
// stays that of the long-row kernel.  Row-level values combine in two
// stages: a warp collective (REDUX / CREDUX / shuffle scan) and a
// shared-memory exchange of the W warp results behind one __syncthreads per
// reduction (double-buffered slots, so no second barrier is needed before the
// next step overwrites them).  Every thread ends up with the row's value, so
// the general search code (row_body: exact and early-stop loops, every exit
// rule, traces, the fill branch) runs unchanged on BlockRow.  Each warp
// streams its slice of the next row into a shared-memory slot with cp.async
// while the current row is searched; selected (value, index) pairs are
// staged in shared memory up to position k and written by the whole CTA.
#pragma once

#include "rtk_kernels.cuh"

namespace rtk {

// Shared-memory exchange slots of the block reductions (one set per CTA).
__device__ __forceinline__ int* block_part_i() {
    __shared__ int part[2][32];
    return &part[0][0];
}
__device__ __forceinline__ float* block_part_f() {
    __shared__ float part[2][32];
    return &part[0][0];
}

template <int E, int W, bool MASKED>
struct BlockRow {
    using Tile = LaneRow<E, true, false>;  // per-warp slice layout (slot strides, masking per slice)
    static constexpr bool kStaged = true;
    static constexpr bool kBlock = true;
    static constexpr int kPad = 0;
    Tile tile;
    mutable unsigned phase = 0;

    __device__ __forceinline__ static int tid() { return (int)threadIdx.x; }
    __device__ __forceinline__ static int warp() { return (int)(threadIdx.x >> 5); }

    // elements of this thread that are real (the row ends at m)
    __device__ __forceinline__ static int lane_valid(int m, int) {
        return MASKED ? max(0, min(E, m - tid() * E)) : E;
    }
    __device__ __forceinline__ void lane_min_max(int m, int, float& mn, float& mx) const {
        tile.lane_min_max(m - warp() * 32 * E, tid() & 31, mn, mx);
    }
    __device__ __forceinline__ int lane_count_ge(float t) const { return tile.lane_count_ge(t); }

    // Sum of the W warp values of an int (every thread gets the total).
    __device__ __forceinline__ int block_sum(int warp_val) const {
        int* part = block_part_i() + 32 * phase;
        phase ^= 1u;
        if ((tid() & 31) == 0) part[warp()] = warp_val;
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) tot += part[i];
        return tot;
    }
    // Exclusive prefix over warps (sum of the warp values of warps < mine) and total.
    __device__ __forceinline__ int block_excl(int warp_val, int& total) const {
        int* part = block_part_i() + 32 * phase;
        phase ^= 1u;
        if ((tid() & 31) == 0) part[warp()] = warp_val;
        __syncthreads();
        int pre = 0, tot = 0;
        const int w = warp();
#pragma unroll
        for (int i = 0; i < W; ++i) {
            pre += i < w ? part[i] : 0;
            tot += part[i];
        }
        total = tot;
        return pre;
    }

    // biased row count (kCountBias + #{v >= t}) from biased lane counts
    __device__ __forceinline__ int count(int lane_biased) const {
        return block_sum(warp_count(lane_biased) - kCountBias) + kCountBias;
    }

    __device__ __forceinline__ void reduce_min_max(float mnl, float mxl, float& mn0, float& mx0) const {
        const float wmn = warp_min_nan(mnl), wmx = warp_max(mxl);
        float* part = block_part_f() + 32 * phase;
        phase ^= 1u;
        if ((tid() & 31) == 0) {
            part[warp()] = wmn;
            part[16 + warp()] = wmx;
        }
        __syncthreads();
        mn0 = part[0];
        mx0 = part[16];
#pragma unroll
        for (int i = 1; i < W; ++i) {
            mn0 = fmin_nan(mn0, part[i]);
            mx0 = fmaxf(mx0, part[16 + i]);
        }
    }

    // First k elements (ascending index) with v >= t staged as (value, index)
    // pairs (the caller guarantees #{v >= t} >= k).
    __device__ __forceinline__ unsigned select_ge(float t, int k, unsigned sbase, int, int lane_hits) const {
        const unsigned cl = (unsigned)lane_hits;
        const unsigned incl = warp_incl_scan(cl);
        const unsigned wtot = __shfl_sync(kFull, incl, 31);
        int total;
        const unsigned pre = (unsigned)block_excl((int)wtot, total);
        unsigned pos = pre + incl - cl;
        const int i0 = tid() * E;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const bool hit = tile.v[q] >= t;
            if (hit && pos < (unsigned)k) stage_put(sbase + 8u * pos, tile.v[q], i0 + q);
            pos += hit ? 1u : 0u;
        }
        return 0u;
    }

    // All v >= t plus the first `need` elements of [lo, t), ascending index
    // (_kernels.py:126-145); counts packed 16 + 16 bits (a row has <= 8192).
    __device__ __forceinline__ void select_fill(float t, float lo, int need, int k, unsigned sbase, int) const {
        unsigned packed = 0;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const bool pa = tile.v[q] >= t;
            const bool pb = (lo <= tile.v[q]) && (tile.v[q] < t);
            packed += (pa ? 1u : 0u) + (pb ? 0x10000u : 0u);
        }
        const unsigned incl = warp_incl_scan(packed);
        const unsigned wtot = __shfl_sync(kFull, incl, 31);
        int total;
        const unsigned pre = (unsigned)block_excl((int)wtot, total);
        const unsigned excl = pre + incl - packed;
        int ea = (int)(excl & 0xffffu), eb = (int)(excl >> 16);
        const int i0 = tid() * E;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const float x = tile.v[q];
            if (x >= t) {
                const int pos = ea + min(eb, need);
                if (pos < k) stage_put(sbase + 8u * pos, x, i0 + q);
                ++ea;
            } else if (lo <= x && x < t) {
                if (eb < need && ea + eb < k) stage_put(sbase + 8u * (ea + eb), x, i0 + q);
                ++eb;
            }
        }
    }

    // The whole CTA writes the k staged pairs.
    __device__ __forceinline__ static void flush_block(unsigned sbase, int k, float* __restrict__ ov,
                                                       int* __restrict__ oi) {
        __syncthreads();
#pragma unroll 1
        for (int j = tid(); j < k; j += W * 32) {
            float v;
            int i;
            stage_get(sbase + 8u * j, v, i);
            ov[j] = v;
            oi[j] = i;
        }
        __syncthreads();
    }
};

// E = 32: caps registers at ~85; wider tiles: about E + 64 registers.
template <int W, int E>
struct BlockMinCtas {
    static constexpr int raw = E <= 32 ? 768 / (W * 32) : 65536 / (W * 32 * (E + 64));
    static constexpr int value = raw > 0 ? raw : 1;
};

// Persistent loop over rows (CTA per row).  Shared memory: k staged pairs,
// then one cp.async slot per warp for its slice of the next row (padding
// chunks NaN-filled once, as in the long-row kernel).
template <int MODE, int W, int E, bool TRACES>
__global__ void __launch_bounds__(W * 32, BlockMinCtas<W, E>::value) rowtopk_block_kernel(Args a) {
    using Row = BlockRow<E, W, true>;
    using Tile = typename Row::Tile;
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int w = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned base = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned sbase = base;
    const unsigned stage_bytes = (8u * (unsigned)a.k + 15u) & ~15u;
    const unsigned slot = base + stage_bytes + (unsigned)w * Tile::kRowBytes;
    const unsigned long long n = (unsigned long long)a.n;
    unsigned r = blockIdx.x;
    if (r >= n) return;
    const unsigned ldx_b = (unsigned)a.ldx * 4u;
    const int mw = a.m - w * 32 * E;  // columns of the row from this warp's slice on
    const bool fp = a.eps_rel == 0.0;
    Tile::fill_slot_nan(slot, lane);
    __syncwarp();
    Tile::stage_async(row_ptr(a.x, r, ldx_b) + w * 32 * E, mw, lane, slot);
    cp_async_commit();
    Row row;
    for (;;) {
        cp_async_wait<0>();
        __syncwarp();  // chunks land in their owner lanes' parts of the slot
        row.tile.load_smem_prefilled(slot, lane);
        const unsigned long long rn = (unsigned long long)r + gridDim.x;
        process_row<MODE, TRACES>(row, r, a, lane, sbase, fp, [&](unsigned tok) {
            __syncwarp();  // every lane has read its part of the slot
            const unsigned salt = tok & a.opaque_zero;
            if (rn < n)
                Tile::stage_async(row_ptr(a.x, (unsigned)rn + salt, ldx_b) + w * 32 * E, mw, lane, slot, salt);
            cp_async_commit();
        });
        if (rn >= n) break;
        r = (unsigned)rn;
    }
    cp_async_wait<0>();
}

}  // namespace rtk
