// rtk_pair.cuh -- paired-row persistent kernel (the hot path).
//
// Each warp processes its rows two at a time (rows r and r + nw of the
// grid-stride sequence) in lockstep: the two rows' min/max reductions,
// bisection steps, selection scans and output flushes are independent
// dependency chains issued back to back, so one row's REDUX / SHFL / LDS
// latency is covered by the other row's instructions.  The selection needs
// one warp scan for both rows (lane hit counts packed 16 + 16 bits).  In
// exact mode the pair loop runs until either row meets cnt == k; the other
// row finishes its search alone (exact_loop_fast), so no step is spent on a
// finished row.  The next pair is prefetched into a second pair of register
// tiles once the current pair has been read (see rowtopk_kernel).
//
// Used for launches without traces on the lane-contiguous register tile
// (M <= 256 here, M % 4 == 0, 16-byte aligned rows; the paired long-row
// kernels of rtk_big.cuh reuse process_pair for 256 < M <= 1024) in
// early-stop mode and in exact mode with eps_rel == 0.  Rows that cannot take
// the fast loop (degenerate, |min| or |max| >= 2^126, NaN) and unpaired last
// rows run the general per-row path (row_body).  Outputs are those of
// rowtopk_kernel.  Both rows' midpoints are one FADD2 + FMUL2 and both rows'
// compare sums one f32x2 tree (mid_fast2, lane_count_ge2).
#pragma once

#include "rtk_kernels.cuh"

namespace rtk {

#ifndef RTK_PAIR_MIN_CTAS
#define RTK_PAIR_MIN_CTAS 2  // __launch_bounds__ min CTAs per SM (caps registers at 64)
#endif
#ifndef RTK_PAIR_MIN_CTAS_E4
#define RTK_PAIR_MIN_CTAS_E4 2  // the same for E = 4 (M <= 128)
#endif
template <int E>
struct PairMinCtas {
    static constexpr int value = E <= 4 ? RTK_PAIR_MIN_CTAS_E4 : RTK_PAIR_MIN_CTAS;
};

// Inclusive warp prefix sum (SHFL.UP's in-range predicate guards the add);
// not volatile, so the compiler may schedule other work between the steps.
__device__ __forceinline__ unsigned warp_incl_scan_nv(unsigned x) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm("{.reg .pred p; .reg .b32 t;\n\t"
            "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
            "@p add.u32 %0, %0, t;}"
            : "+r"(x)
            : "r"(d));
    return x;
}

// mid_fast of two brackets at once: one FADD2 + one FMUL2 (IEEE round to
// nearest per half, subnormals kept: bit-identical to two mid_fast calls).
__device__ __forceinline__ void mid_fast2(float mnA, float mxA, float mnB, float mxB, float& midA, float& midB) {
    asm("{.reg .b64 p, q; mov.b64 p, {%2, %3}; mov.b64 q, {%4, %5}; add.rn.f32x2 p, p, q;"
        " mul.rn.f32x2 p, p, %6; mov.b64 {%0, %1}, p;}"
        : "=f"(midA), "=f"(midB)
        : "f"(mnA), "f"(mnB), "f"(mxA), "f"(mxB), "l"(0x3f0000003f000000ull));
}

// Biased lane counts of both rows of a pair (A.v >= tA, B.v >= tB): the
// compare results of element q of A and B form one f32x2 pair, so the sum
// tree is E FADD2 (with the 2^23 bias) for both rows.
template <class Row>
__device__ __forceinline__ void lane_count_ge2(const Row& A, const Row& B, float tA, float tB, int& lA, int& lB) {
    constexpr int E = Row::kSlots;
    static_assert(E % 4 == 0, "pair count tree needs E % 4 == 0");
    float xa[E / 2], xb[E / 2];
#pragma unroll
    for (int q = 0; q < E; q += 2) {
        xa[q / 2] = set_ge(A.v[q], tA);
        xb[q / 2] = set_ge(B.v[q], tB);
        add2(xa[q / 2], xb[q / 2], set_ge(A.v[q + 1], tA), set_ge(B.v[q + 1], tB));
    }
#pragma unroll
    for (int w = 1; w < E / 2; w *= 2)
#pragma unroll
        for (int q = 0; q + w < E / 2; q += 2 * w) add2(xa[q], xb[q], xa[q + w], xb[q + w]);
    add2(xa[0], xb[0], 0x1p23f, 0x1p23f);
    lA = __float_as_int(xa[0]);
    lB = __float_as_int(xb[0]);
}

// Both rows selected at thresholds tA, tB with biased lane hit counts hA, hB
// (#{v >= t} per lane): stage row copies and indices, then write the first k
// (value, index) pairs of each row.
template <class Row>
__device__ __forceinline__ void select_flush_pair(const Row& A, const Row& B, float tA, float tB, int hA, int hB,
                                                  unsigned sA, unsigned sB, int lane, int k, float* __restrict__ ovA,
                                                  int* __restrict__ oiA, float* __restrict__ ovB,
                                                  int* __restrict__ oiB, bool vec4) {
    A.stage_row(sA, lane);
    B.stage_row(sB, lane);
    const unsigned packed = (unsigned)(hA - (int)kLaneBias) | ((unsigned)(hB - (int)kLaneBias) << 16);
    const unsigned excl = warp_incl_scan_nv(packed) - packed;
    A.stage_idx(tA, sA, lane, excl & 0xffffu);
    B.stage_idx(tB, sB, lane, excl >> 16);
    __syncwarp();
    if (k <= 32) {
        if (lane < k) {
            int iA, iB;
            float xA, xB;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(iA) : "r"(sA + Row::kIdxOff + 4u * lane) : "memory");
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(iB) : "r"(sB + Row::kIdxOff + 4u * lane) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xA) : "r"(Row::copy_addr(sA, Row::clamp_slot(iA))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xB) : "r"(Row::copy_addr(sB, Row::clamp_slot(iB))) : "memory");
            ovA[lane] = xA;
            oiA[lane] = iA;
            ovB[lane] = xB;
            oiB[lane] = iB;
        }
        __syncwarp();
        return;
    }
    if (vec4) {  // 4 consecutive outputs per lane: LDS.128 of indices, STG.128 stores
#pragma unroll 1
        for (int j = 4 * lane; j < k; j += 128) {
            int4 iA, iB;
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(iA.x), "=r"(iA.y), "=r"(iA.z), "=r"(iA.w)
                         : "r"(sA + Row::kIdxOff + 4u * j)
                         : "memory");
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(iB.x), "=r"(iB.y), "=r"(iB.z), "=r"(iB.w)
                         : "r"(sB + Row::kIdxOff + 4u * j)
                         : "memory");
            float4 xA, xB;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xA.x) : "r"(Row::copy_addr(sA, Row::clamp_slot(iA.x))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xA.y) : "r"(Row::copy_addr(sA, Row::clamp_slot(iA.y))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xA.z) : "r"(Row::copy_addr(sA, Row::clamp_slot(iA.z))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xA.w) : "r"(Row::copy_addr(sA, Row::clamp_slot(iA.w))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xB.x) : "r"(Row::copy_addr(sB, Row::clamp_slot(iB.x))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xB.y) : "r"(Row::copy_addr(sB, Row::clamp_slot(iB.y))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xB.z) : "r"(Row::copy_addr(sB, Row::clamp_slot(iB.z))) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xB.w) : "r"(Row::copy_addr(sB, Row::clamp_slot(iB.w))) : "memory");
            *reinterpret_cast<float4*>(ovA + j) = xA;
            *reinterpret_cast<int4*>(oiA + j) = iA;
            *reinterpret_cast<float4*>(ovB + j) = xB;
            *reinterpret_cast<int4*>(oiB + j) = iB;
        }
        __syncwarp();
        return;
    }
#pragma unroll 1
    for (int j = lane; j < k; j += 32) {
        int iA, iB;
        float xA, xB;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(iA) : "r"(sA + Row::kIdxOff + 4u * j) : "memory");
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(iB) : "r"(sB + Row::kIdxOff + 4u * j) : "memory");
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xA) : "r"(Row::copy_addr(sA, Row::clamp_slot(iA))) : "memory");
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xB) : "r"(Row::copy_addr(sB, Row::clamp_slot(iB))) : "memory");
        ovA[j] = xA;
        oiA[j] = iA;
        ovB[j] = xB;
        oiB[j] = iB;
    }
    __syncwarp();
}

// Selection of both rows at thresholds tA, tB (biased lane hits hA, hB):
// LaneRow tiles share one packed scan and the row-copy flush
// (select_flush_pair); the long-row tiles (LaneRowCut, paired TMA kernel)
// stage each row's first k pairs and flush them.
template <class Row>
__device__ __forceinline__ void select_two(const Row& A, const Row& B, float tA, float tB, int hA, int hB, unsigned sA,
                                           unsigned sB, int lane, int k, float* __restrict__ ovA, int* __restrict__ oiA,
                                           float* __restrict__ ovB, int* __restrict__ oiB, bool vec4, unsigned oz) {
    if constexpr (Row::kPad > 0) {
        select_flush_pair(A, B, tA, tB, hA, hB, sA, sB, lane, k, ovA, oiA, ovB, oiB, vec4);
    } else {
        const unsigned dA = A.select_ge(tA, k, sA, lane, hA - (int)kLaneBias);
        const unsigned dB = B.select_ge(tB, k, sB, lane, hB - (int)kLaneBias);
        flush_staged<Row>(sA, k, ovA, oiA, lane, dA & oz);
        flush_staged<Row>(sB, k, ovB, oiB, lane, dB & oz);
    }
}

// Exact mode, one row after its fast loop ended (eq: cnt == k at mid).
template <class Row>
__device__ __forceinline__ void finish_exact(const Row& row, const Args& a, int lane, unsigned sbase, bool eq,
                                             float mn, float mx, float mid, int cnt, int it, int lc,
                                             float* __restrict__ ov, int* __restrict__ oi) {
    const int kb = a.k + kCountBias;
    if (eq) {
        row.select_ge(mid, a.k, sbase, lane, lc - (int)kLaneBias);
        flush_staged<Row>(sbase, a.k, ov, oi, lane);
        return;
    }
    float thres = mid;
    int reason;
    if (it >= a.hard_cap)
        reason = kExitHardCapReached;  // selection treats HARD_CAP and IBE alike
    else
        reason = exact_loop<true, true>(row, kb, 0.0, a.hard_cap, mn, mx, thres, cnt, it, lc);
    select_exact(row, a, lane, sbase, true, reason, thres, mn, mx, cnt, lc, ov, oi);
}

// ------------------------------------------------------- fused MaxK rows
//
// rtk_maxk_dense: after a row's selection (k indices staged at
// sbase + kIdxOff by every path: select_flush_pair, finish_exact, row_body),
// write the dense MaxK row -- x with all but the selected entries set to
// +0 -- and / or a uint8 copy of the indices (the compact index layout of
// the MaxK sparse rows for M <= 256), straight from the register tile: the
// staged indices set bits of a 32E-bit shared bitmap (atomic OR), then each
// lane stores its E contiguous
// elements (value or zero) with vector stores in the input type (16-bit
// rows: the tile holds their exact fp32 widening, narrowed back exactly).
// Replaces the select -> scatter_rows pair (one launch and the N*k*8-byte
// values/indices round trip fewer for the dense consumer).
template <class Row>
struct DenseBitmap {
    static constexpr unsigned kBytes = (4u * Row::kSlots + 15u) & ~15u;  // 32E bits, 16-byte padded
};

template <class In, class Row>
__device__ __forceinline__ void dense_row(const Row& R, unsigned sbase, const Args& a, unsigned r, int lane) {
    constexpr int E = Row::kSlots;
    static_assert(E == 4 || E == 8, "fused MaxK rows: E = 4 or 8 (M = 128 or 256)");
    if (a.idx8) {  // uint8 copy of the staged indices (M <= 256)
        unsigned char* o8 = a.idx8 + (unsigned long long)r * (unsigned long long)a.ld8;
        for (int j = lane; j < a.k; j += 32) {
            unsigned i;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(i) : "r"(sbase + Row::kIdxOff + 4u * j) : "memory");
            o8[j] = (unsigned char)i;
        }
    }
    if (!a.dense) return;
    const unsigned bm = sbase + Row::kStageBytes;
    if (lane < E) asm volatile("st.shared.b32 [%0], %1;" ::"r"(bm + 4u * lane), "r"(0u) : "memory");
    __syncwarp();
    for (int j = lane; j < a.k; j += 32) {
        unsigned i;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(i) : "r"(sbase + Row::kIdxOff + 4u * j) : "memory");
        i &= 32u * E - 1u;  // NaN rows (reported, output unspecified) may stage garbage
        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(bm + 4u * (i >> 5)), "r"(1u << (i & 31u)) : "memory");
    }
    __syncwarp();
    unsigned w;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(bm + 4u * ((unsigned)(lane * E) >> 5)) : "memory");
    const unsigned bits = w >> ((unsigned)(lane * E) & 31u);
    float o[E];
#pragma unroll
    for (int q = 0; q < E; ++q) o[q] = (bits >> q) & 1u ? R.v[q] : 0.0f;
    In* dp = row_ptr(reinterpret_cast<In*>(a.dense), r, (unsigned)(a.ldd * (long long)sizeof(In))) + lane * E;
    if constexpr (std::is_same<In, float>::value) {
#pragma unroll
        for (int g = 0; g < E / 4; ++g)
            __stcs(reinterpret_cast<float4*>(dp + 4 * g), make_float4(o[4 * g], o[4 * g + 1], o[4 * g + 2], o[4 * g + 3]));
    } else {
        unsigned h[E / 2];
#pragma unroll
        for (int q = 0; q < E / 2; ++q) {
            In lo, hi;
            if constexpr (std::is_same<In, __nv_bfloat16>::value) {
                lo = __float2bfloat16_rn(o[2 * q]);
                hi = __float2bfloat16_rn(o[2 * q + 1]);
            } else {
                lo = __float2half_rn(o[2 * q]);
                hi = __float2half_rn(o[2 * q + 1]);
            }
            h[q] = (unsigned)*reinterpret_cast<unsigned short*>(&lo) |
                   ((unsigned)*reinterpret_cast<unsigned short*>(&hi) << 16);
        }
        if constexpr (E == 8)
            __stcs(reinterpret_cast<uint4*>(dp), make_uint4(h[0], h[1], h[2], h[3]));
        else
            __stcs(reinterpret_cast<uint2*>(dp), make_uint2(h[0], h[1]));
    }
    __syncwarp();  // the bitmap and the staging are reused by the next row
}

// Row r of the input into a register tile: fp32 rows as they are, 16-bit
// rows (In = __nv_bfloat16 / __half, rtk_rowtopk_x16) widened on load.
template <class In, class Row>
__device__ __forceinline__ void load_tile(Row& R, const Args& a, unsigned r, unsigned ldx_b, int lane) {
    if constexpr (std::is_same<In, float>::value)
        R.load(row_ptr(a.x, r, ldx_b), a.m, lane);
    else
        R.template load16<In>(row_ptr(reinterpret_cast<const In*>(a.x), r, ldx_b), a.m, lane);
}

// ------------------------------------ exact mode, long rows: candidate set
//
// For the paired long-row kernels (LaneRowCut tiles, E = 12..32) the exact
// search runs in two phases.  Full phase: reference bisection steps counting
// the whole tile, until the count at the bracket's lower end mn is at most
// the candidate capacity 32 C (or cnt == k).  Every later midpoint is >= mn,
// so counting the candidate set S = {v >= mn} gives the reference's count;
// S is staged as (value, index) pairs in index order (one packed warp scan
// for both rows) and read back C slots per lane.  Candidate phase: the same
// reference steps (same midpoints, same decisions) on S -- C compares per
// lane instead of E.  Selection: S at the final midpoint (cnt == k) by one
// ballot prefix per slot, written straight to the output row.  A row meeting
// cnt == k in the full phase stages S = {v >= mid} (k entries) and takes the
// same selection; rows out of fast steps (stuck / tied) finish on the general
// path (the tile is re-read).  At E = 8 (M = 256) the staging costs more than
// the cheaper steps save (measured); at E >= 12 a full step costs 1.5 E + 13
// instructions per row and a candidate step about 15.
#ifndef RTK_LONG_CAND
#define RTK_LONG_CAND 1
#endif
// candidate slots per lane: 2 (k <= 40), 4 (k <= 96), 8 (k <= 192; E >= 16,
// in a separate kernel instantiation (CMAX = 8): compiled into the k <= 96
// kernels the third search raised their spills).  At E = 16 a candidate step
// still counts half the tile, and measured 4-6% faster at M = 512.
#ifndef RTK_CAND8_MIN_E
#define RTK_CAND8_MIN_E 16
#endif
#ifndef RTK_CAND2_KMAX  // switch points measured against 52 / 96 and 32 / 72: best or equal on 12 shapes
#define RTK_CAND2_KMAX 40
#endif
#ifndef RTK_CAND4_KMAX
#define RTK_CAND4_KMAX 96
#endif
template <int E>
__host__ __device__ constexpr bool long_cand8(int k) {
    return E >= RTK_CAND8_MIN_E && k > RTK_CAND4_KMAX && k <= 192;
}
// staging bytes per row of the paired long-row kernels: the k-pair staging
// of LaneRowCut or the candidate set, whichever is larger
template <class Row>
__host__ __device__ constexpr unsigned pair_stage_bytes(int k) {
    const int slots = k <= RTK_CAND2_KMAX ? 2 : (k <= RTK_CAND4_KMAX ? 4 : (long_cand8<Row::kSlots>(k) ? 8 : 0));
    const unsigned cand = 8u * 32u * (unsigned)slots;
    return Row::stage_bytes(k) > cand ? Row::stage_bytes(k) : cand;
}

template <int C>
struct CandSet {
    float v[C];
    int i[C];
};

// Stage this lane's elements with v >= t as (value, index) pairs at entries
// excl, excl + 1, ... of the list at sbase.
template <class Row>
__device__ __forceinline__ void stage_cand(const Row& R, float t, unsigned sbase, int lane, unsigned excl) {
    constexpr int E = Row::kSlots;
    unsigned addr = sbase + 8u * excl;
    const int i0 = lane * E;
#pragma unroll
    for (int q = 0; q < E; ++q) {
        if (R.v[q] >= t) {
            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(__float_as_int(R.v[q])), "r"(i0 + q)
                         : "memory");
            addr += 8u;
        }
    }
}

// Entries j = lane + 32 q of the staged list (ns of them); past ns: NaN.
template <int C>
__device__ __forceinline__ void load_cand(unsigned sbase, int lane, int ns, CandSet<C>& S) {
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const int j = lane + 32 * q;
        int x, i;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(i) : "r"(sbase + 8u * j) : "memory");
        S.i[q] = i;
        S.v[q] = j < ns ? __int_as_float(x) : __int_as_float(0x7fffffff);
    }
}

// Biased lane counts of both rows' candidates >= tA / tB (one FADD2 per slot).
template <int C>
__device__ __forceinline__ void cand_count2(const CandSet<C>& SA, const CandSet<C>& SB, float tA, float tB, int& lA,
                                            int& lB) {
    float xa = 0x1p23f, xb = 0x1p23f;
#pragma unroll
    for (int q = 0; q < C; ++q) add2(xa, xb, set_ge(SA.v[q], tA), set_ge(SB.v[q], tB));
    lA = __float_as_int(xa);
    lB = __float_as_int(xb);
}

template <int C>
__device__ __forceinline__ void cand_steps_alone(const CandSet<C>& S, int kb, int steps, float& mn, float& mx,
                                                 float& mid, int& c, int& it) {
#pragma unroll 1
    while (c != kb && it < steps) {
        ++it;
        mid = mid_fast(mn, mx);
        float x = 0x1p23f;
#pragma unroll
        for (int q = 0; q < C; ++q) x = __fadd_rn(x, set_ge(S.v[q], mid));
        c = warp_count(__float_as_int(x));
        const bool lt = c < kb;
        mx = lt ? mid : mx;
        mn = lt ? mn : mid;
    }
}

// Full-phase steps of one row until cnt == k, the count at mn is <= the
// capacity (clb, hl: biased row / lane counts at mn), or `steps`.
template <class Row>
__device__ __forceinline__ void full_steps_alone(const Row& R, int kb, int capb, int steps, float& mn, float& mx,
                                                 float& mid, int& c, int& l, int& hl, int& clb, int& it) {
#pragma unroll 1
    while (c != kb && clb > capb && it < steps) {
        ++it;
        mid = mid_fast(mn, mx);
        l = R.lane_count_ge(mid);
        c = warp_count(l);
        const bool lt = c < kb;
        mx = lt ? mid : mx;
        mn = lt ? mn : mid;
        hl = lt ? hl : l;
        clb = lt ? clb : c;
    }
}

// The candidates >= t (exactly k of them) in index order, to the output row.
template <int C>
__device__ __forceinline__ void emit_cand(const CandSet<C>& S, float t, float* __restrict__ ov,
                                          int* __restrict__ oi) {
    const unsigned lt = lanemask_lt();
    int base = 0;
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const bool p = S.v[q] >= t;
        const unsigned b = __ballot_sync(kFull, p);
        const int pos = base + __popc(b & lt);
        if (p) {
            ov[pos] = S.v[q];
            oi[pos] = S.i[q];
        }
        base += __popc(b);
    }
}

template <int C, class In, class Row>
__device__ __forceinline__ void exact_pair_cand(const Row& A, const Row& B, unsigned rA, unsigned rB, const Args& a,
                                                int lane, unsigned sA, unsigned sB, int steps, float mnA, float mxA,
                                                float mnB, float mxB, float* __restrict__ ovA, int* __restrict__ oiA,
                                                float* __restrict__ ovB, int* __restrict__ oiB) {
    const int k = a.k;
    const int kb = k + kCountBias;
    const int capb = 32 * C + kCountBias;
    float midA, midB;
    int cA, cB, lA, lB, it = 0;
    int hA = (int)kLaneBias + Row::lane_valid(a.m, lane), hB = hA;  // lane counts at mn
    int clA = a.m + kCountBias, clB = clA;                          // row counts at mn
#pragma unroll 1
    do {
        ++it;
        mid_fast2(mnA, mxA, mnB, mxB, midA, midB);
        lane_count_ge2(A, B, midA, midB, lA, lB);
        cA = warp_count(lA);
        cB = warp_count(lB);
        const bool ltA = cA < kb, ltB = cB < kb;
        mxA = ltA ? midA : mxA;
        mnA = ltA ? mnA : midA;
        hA = ltA ? hA : lA;
        clA = ltA ? clA : cA;
        mxB = ltB ? midB : mxB;
        mnB = ltB ? mnB : midB;
        hB = ltB ? hB : lB;
        clB = ltB ? clB : cB;
    } while (cA != kb && cB != kb && clA > capb && clB > capb && it < steps);
    int itA = it, itB = it;
    full_steps_alone(A, kb, capb, steps, mnA, mxA, midA, cA, lA, hA, clA, itA);
    full_steps_alone(B, kb, capb, steps, mnB, mxB, midB, cB, lB, hB, clB, itB);
    bool eqA = cA == kb, eqB = cB == kb;
    if (!((eqA || clA <= capb) && (eqB || clB <= capb))) {  // out of fast steps (cold)
        finish_exact(A, a, lane, sA, eqA, mnA, mxA, midA, cA, itA, lA, ovA, oiA);
        finish_exact(B, a, lane, sB, eqB, mnB, mxB, midB, cB, itB, lB, ovB, oiB);
        return;
    }
    // S = {v >= T} of both rows (T = mid on cnt == k, else mn)
    const float tA = eqA ? midA : mnA, tB = eqB ? midB : mnB;
    const int nA = eqA ? k : clA - kCountBias, nB = eqB ? k : clB - kCountBias;
    const unsigned HA = (unsigned)((eqA ? lA : hA) - (int)kLaneBias), HB = (unsigned)((eqB ? lB : hB) - (int)kLaneBias);
    const unsigned packed = HA | (HB << 16);
    const unsigned excl = warp_incl_scan_nv(packed) - packed;
    stage_cand(A, tA, sA, lane, excl & 0xffffu);
    stage_cand(B, tB, sB, lane, excl >> 16);
    __syncwarp();
    CandSet<C> SA, SB;
    load_cand(sA, lane, nA, SA);
    load_cand(sB, lane, nB, SB);
    __syncwarp();
    if (!eqA && !eqB && itA < steps && itB < steps) {  // (the full phase may have used up the steps)
#pragma unroll 1
        do {
            ++itA;
            ++itB;
            mid_fast2(mnA, mxA, mnB, mxB, midA, midB);
            int lcA, lcB;
            cand_count2(SA, SB, midA, midB, lcA, lcB);
            cA = warp_count(lcA);
            cB = warp_count(lcB);
            const bool ltA = cA < kb, ltB = cB < kb;
            mxA = ltA ? midA : mxA;
            mnA = ltA ? mnA : midA;
            mxB = ltB ? midB : mxB;
            mnB = ltB ? mnB : midB;
        } while (cA != kb && cB != kb && itA < steps && itB < steps);  // the rows' counts differ after the full phase
    }
    cand_steps_alone(SA, kb, steps, mnA, mxA, midA, cA, itA);
    cand_steps_alone(SB, kb, steps, mnB, mxB, midB, cB, itB);
    eqA = cA == kb;
    eqB = cB == kb;
    if (eqA && eqB) {
        emit_cand(SA, midA, ovA, oiA);
        emit_cand(SB, midB, ovB, oiB);
        return;
    }
    // out of fast steps in the candidate phase (cold): the general path on a
    // re-read tile
    const unsigned ldx_b = (unsigned)a.ldx * (unsigned)sizeof(In);
    if (eqA) {
        emit_cand(SA, midA, ovA, oiA);
    } else {
        Row T;
        load_tile<In>(T, a, rA, ldx_b, lane);
        finish_exact(T, a, lane, sA, false, mnA, mxA, midA, cA, itA, T.lane_count_ge(midA), ovA, oiA);
    }
    if (eqB) {
        emit_cand(SB, midB, ovB, oiB);
    } else {
        Row T;
        load_tile<In>(T, a, rB, ldx_b, lane);
        finish_exact(T, a, lane, sB, false, mnB, mxB, midB, cB, itB, T.lane_count_ge(midB), ovB, oiB);
    }
}

// mn0 < mx0 with both inside (-2^126, 2^126): non-degenerate (both modes),
// finite (exact mode's eps_rel == 0 loop test) and overflow-free midpoints.
// NaN compares false.
__device__ __forceinline__ bool fast_eligible(float mn0, float mx0) {
    return mx0 > mn0 && mn0 > -0x1p126f && mx0 < 0x1p126f;
}

// One pair of rows (rA = r, rB = r + nw when hasB).  `after_load(token)`
// issues the next pair's loads once both tiles have been read.
template <int MODE, class In, int CMAX, class Row, class Hook>
__device__ __forceinline__ void process_pair_sel(const Row& A, const Row& B, unsigned rA, unsigned rB, bool hasB,
                                                 const Args& a, int lane, unsigned sA, unsigned sB, int steps,
                                                 const Hook& after_load) {
    float mnlA, mxlA, mnlB, mxlB;
    A.lane_min_max(a.m, lane, mnlA, mxlA);
    B.lane_min_max(a.m, lane, mnlB, mxlB);
    after_load(__float_as_uint(mnlA) ^ __float_as_uint(mxlB));
    const float mn0A = warp_min_nan(mnlA), mx0A = warp_max(mxlA);
    const float mn0B = warp_min_nan(mnlB), mx0B = warp_max(mxlB);
    if (mn0A != mn0A) report_nan(a.nan_row, rA, lane);
    if (hasB && mn0B != mn0B) report_nan(a.nan_row, rB, lane);
    const unsigned ldo_b = (unsigned)a.ldo * 4u;
    float* ovA = row_ptr(a.vals, rA, ldo_b);
    int* oiA = row_ptr(a.idx, rA, ldo_b);
    float* ovB = row_ptr(a.vals, rB, ldo_b);
    int* oiB = row_ptr(a.idx, rB, ldo_b);
    const int k = a.k;
    const int kb = k + kCountBias;

    if (!(hasB && fast_eligible(mn0A, mx0A) && fast_eligible(mn0B, mx0B))) {
        row_body<MODE, false>(A, rA, a, lane, sA, true, mn0A, mx0A);
        if (hasB) row_body<MODE, false>(B, rB, a, lane, sB, true, mn0B, mx0B);
        return;
    }

    float mnA = mn0A, mxA = mx0A, mnB = mn0B, mxB = mx0B;
    if constexpr (MODE == kEarly) {
        // Algorithm 2 (_kernels.py:96-102) on both rows; lane counts at mn
        int hA = (int)kLaneBias + Row::lane_valid(a.m, lane), hB = hA;
#pragma unroll 1
        for (int i = 0; i < steps; ++i) {
            float midA, midB;
            mid_fast2(mnA, mxA, mnB, mxB, midA, midB);
            int lA, lB;
            lane_count_ge2(A, B, midA, midB, lA, lB);
            const bool ltA = warp_count(lA) < kb, ltB = warp_count(lB) < kb;
            mxA = ltA ? midA : mxA;
            mnA = ltA ? mnA : midA;
            hA = ltA ? hA : lA;
            mxB = ltB ? midB : mxB;
            mnB = ltB ? mnB : midB;
            hB = ltB ? hB : lB;
        }
        // first k indices with v >= mn (_kernels.py:205-212)
        // (scalar flush: the vectorised one measured 2% slower in early-stop mode)
        select_two(A, B, mnA, mnB, hA, hB, sA, sB, lane, k, ovA, oiA, ovB, oiB, false, a.opaque_zero);
    } else {
        if constexpr (RTK_LONG_CAND && Row::kPad == 0) {  // long rows: the candidate-set search above
            if constexpr (CMAX >= 8) {  // launched for long_cand8(k) only
                exact_pair_cand<8, In>(A, B, rA, rB, a, lane, sA, sB, steps, mnA, mxA, mnB, mxB, ovA, oiA, ovB, oiB);
                return;
            } else {
                if (k <= RTK_CAND2_KMAX) {
                    exact_pair_cand<2, In>(A, B, rA, rB, a, lane, sA, sB, steps, mnA, mxA, mnB, mxB, ovA, oiA, ovB,
                                           oiB);
                    return;
                }
                if (k <= RTK_CAND4_KMAX) {
                    exact_pair_cand<4, In>(A, B, rA, rB, a, lane, sA, sB, steps, mnA, mxA, mnB, mxB, ovA, oiA, ovB,
                                           oiB);
                    return;
                }
            }
        }
        // Algorithm 1 fast steps (exact_loop_fast) on both rows until either
        // meets cnt == k; the other continues alone.
        float midA, midB;
        int cA, cB, lA, lB, it = 0;
#pragma unroll 1
        do {
            ++it;
            mid_fast2(mnA, mxA, mnB, mxB, midA, midB);
            lane_count_ge2(A, B, midA, midB, lA, lB);
            cA = warp_count(lA);
            cB = warp_count(lB);
            const bool ltA = cA < kb, ltB = cB < kb;
            mxA = ltA ? midA : mxA;
            mnA = ltA ? mnA : midA;
            mxB = ltB ? midB : mxB;
            mnB = ltB ? mnB : midB;
        } while (cA != kb && cB != kb && it < steps);
        // equality taken once here: as loop-carried flags it cost two
        // predicate instructions per pair-step (measured 2-4% in exact mode)
        bool eqA = cA == kb, eqB = cB == kb;
        int itA = it, itB = it;
        if (!eqA && itA < steps) eqA = exact_loop_fast(A, kb, steps, mnA, mxA, midA, cA, itA, lA);
        if (!eqB && itB < steps) eqB = exact_loop_fast(B, kb, steps, mnB, mxB, midB, cB, itB, lB);
        if (eqA && eqB) {
            select_two(A, B, midA, midB, lA, lB, sA, sB, lane, k, ovA, oiA, ovB, oiB, a.out_vec4 != 0, a.opaque_zero);
        } else {
            finish_exact(A, a, lane, sA, eqA, mnA, mxA, midA, cA, itA, lA, ovA, oiA);
            finish_exact(B, a, lane, sB, eqB, mnB, mxB, midB, cB, itB, lB, ovB, oiB);
        }
    }
}

// The pair's selection, then (DENSE, rtk_maxk_dense) both fused MaxK rows.
template <int MODE, bool DENSE, class In, int CMAX = 4, class Row, class Hook>
__device__ __forceinline__ void process_pair(const Row& A, const Row& B, unsigned rA, unsigned rB, bool hasB,
                                             const Args& a, int lane, unsigned sA, unsigned sB, int steps,
                                             const Hook& after_load) {
    process_pair_sel<MODE, In, CMAX>(A, B, rA, rB, hasB, a, lane, sA, sB, steps, after_load);
    if constexpr (DENSE) {
        dense_row<In>(A, sA, a, rA, lane);
        if (hasB) dense_row<In>(B, sB, a, rB, lane);
    }
}

// Persistent loop over row pairs (r, r + nw), stepping 2 nw; register
// double buffering of the pair (the roles of the two tile pairs alternate
// between the two unrolled halves).  In: the input element type.
// DENSE: also write the fused MaxK rows (rtk_maxk_dense; one bitmap of
// DenseBitmap bytes after each row's staging).
template <int E, bool DENSE>
struct PairStage {
    static constexpr unsigned kRowStride = LaneRow<E, false>::kStageBytes + (DENSE ? DenseBitmap<LaneRow<E, false>>::kBytes : 0u);
    static constexpr unsigned kWarpBytes = 2u * kRowStride;
};

template <int MODE, int E, bool MASKED, bool WIDE, class In = float, bool DENSE = false>
__global__ void __launch_bounds__(RTK_CTA_THREADS, PairMinCtas<E>::value) rowtopk_pair_kernel(Args a) {
    using Row = LaneRow<E, MASKED, WIDE>;
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned wpc = blockDim.x >> 5;
    const unsigned sA = (unsigned)__cvta_generic_to_shared(smem) + (unsigned)wid * PairStage<E, DENSE>::kWarpBytes;
    const unsigned sB = sA + PairStage<E, DENSE>::kRowStride;
    const unsigned nw = gridDim.x * wpc;
    const unsigned n = (unsigned)a.n;  // the host guarantees n + 2 nw < 2^32
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const unsigned last = n - 1;
    const unsigned ldx_b = (unsigned)a.ldx * (unsigned)sizeof(In);
    const unsigned oz = a.opaque_zero;
    const int steps = MODE == kEarly ? a.max_iter : min(a.hard_cap, RTK_FAST_STEPS);
    Row A, B, C, D;
    load_tile<In>(A, a, r, ldx_b, lane);
    load_tile<In>(B, a, min(r + nw, last), ldx_b, lane);
    for (;;) {
        const unsigned rn = r + 2 * nw;
        process_pair<MODE, DENSE, In>(A, B, r, r + nw, r + nw < n, a, lane, sA, sB, steps, [&](unsigned tok) {
            tok &= oz;
            load_tile<In>(C, a, min(rn, last) + tok, ldx_b, lane);
            load_tile<In>(D, a, min(rn + nw, last) + tok, ldx_b, lane);
        });
        if (rn >= n) break;
        r = rn;
        const unsigned rn2 = r + 2 * nw;
        process_pair<MODE, DENSE, In>(C, D, r, r + nw, r + nw < n, a, lane, sA, sB, steps, [&](unsigned tok) {
            tok &= oz;
            load_tile<In>(A, a, min(rn2, last) + tok, ldx_b, lane);
            load_tile<In>(B, a, min(rn2 + nw, last) + tok, ldx_b, lane);
        });
        if (rn2 >= n) break;
        r = rn2;
    }
}

}  // namespace rtk
