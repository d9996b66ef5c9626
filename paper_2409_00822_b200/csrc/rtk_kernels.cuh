// rtk_kernels.cuh -- sm_100a kernels for row-wise top-k by threshold bisection.
//
// One warp owns one row.  The row lives in registers (up to M = 1024 fp32,
// 32 per lane), loaded with 128-bit streaming loads and prefetched one row
// ahead; every bisection step is a per-lane FSET.BF/FADD2 compare-accumulate
// plus one REDUX.SUM, min/max are CREDUX.MIN/MAX.F32 warp reductions, and
// the selection is a warp prefix scan that writes exactly k (value, index)
// pairs in ascending index order.  The launch is a persistent grid-stride
// loop over rows.  Rows with M > 1024 take the same algorithm with the row
// re-read from L1/L2 on each pass (GlobalRow).
//
// Numeric contract (bit-exact with /root/reference/pkg/src/rowtopk/_kernels.py):
//   * all comparisons are fp32 IEEE >= (_kernels.py:43,75-84,120,140,207);
//   * the midpoint equals F32((F64(a)+F64(b))*0.5) (_kernels.py:72,97), here
//     computed in fp32 with an overflow fallback (proven
//     on CPU in tests/test_oracle.py::test_fp32_midpoint_identity_random_bits);
//   * the exact-mode loop test is the float64 `mx - mn > eps_rel*mx0`
//     (_kernels.py:60,65); for eps_rel == 0 it reduces to the fp32
//     `isfinite(mx0) && mx > mn`;
//   * compiled without fast-math, -ftz=false, -fmad=false.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace rtk {

constexpr int kExitCountEqualsK = 1;        // _kernels.py:19
constexpr int kExitIntervalBelowEps = 2;    // _kernels.py:20
constexpr int kExitMaxIterReached = 3;      // _kernels.py:21
constexpr int kExitHardCapReached = 4;      // _kernels.py:22
constexpr int kExitDegenerateRow = 5;       // _kernels.py:23
constexpr unsigned kFull = 0xffffffffu;

enum Mode : int { kExact = 0, kEarly = 1, kTrace = 2 };

#ifndef RTK_MIN_CTAS
#define RTK_MIN_CTAS 1  // __launch_bounds__ min CTAs per SM for the row kernels
#endif
#ifndef RTK_CTA_THREADS
#define RTK_CTA_THREADS 512  // threads per CTA of the row kernels (measured best at M = 256)
#endif

struct Args {
    const float* __restrict__ x;
    long long n;
    int m;
    long long ldx;
    int k;
    double eps_rel;
    int hard_cap;
    int max_iter;
    float* __restrict__ vals;
    int* __restrict__ idx;
    long long ldo;
    int* __restrict__ iters;
    signed char* __restrict__ reasons;
    unsigned* __restrict__ nan_row;
    // Always 0 at run time; ANDed into the next row's load offset so that the
    // load depends on the current row's lane min/max (see rowtopk_kernel).
    unsigned opaque_zero;
    // Output rows take 16-byte stores in the paired kernel's flush: vals / idx
    // 16-byte aligned, ldo % 4 == 0, k % 4 == 0 and k >= 128 (set by the host).
    int out_vec4;
    // Fused MaxK dense output (rtk_maxk_dense, paired kernel only): row r of
    // x with all but the selected entries zeroed, at dense + r * ldd elements
    // of the input type.
    void* dense;
    long long ldd;
    // ... and / or the selected indices as uint8 (M <= 256), row r at idx8 + r * ld8.
    unsigned char* idx8;
    long long ld8;
};

// ---------------------------------------------------------------- scalars

__device__ __forceinline__ float fmin_nan(float a, float b) {
    float d;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// Warp-wide fp32 min (NaN-propagating: a NaN anywhere in the row makes mn0
// NaN) and max, as sm_100 CREDUX.MIN/MAX.F32 into uniform registers.
__device__ __forceinline__ float warp_min_nan(float v) {
    float d;
    asm volatile("redux.sync.min.NaN.f32 %0, %1, 0xffffffff;" : "=f"(d) : "f"(v));
    return d;
}
__device__ __forceinline__ float warp_max(float v) {
    float d;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(d) : "f"(v));
    return d;
}

// 1.0f if a >= b else 0.0f (FSET.BF.GE; NaN compares false).
__device__ __forceinline__ float set_ge(float a, float b) {
    float d;
    asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// (x, y) += (a, b) as one packed FADD2 (sm_100 f32x2).  Sums of 0/1 values
// below 2^23 are exact.
__device__ __forceinline__ void add2(float& x, float& y, float a, float b) {
    asm("{.reg .b64 p, q; mov.b64 p, {%0, %1}; mov.b64 q, {%2, %3}; add.rn.f32x2 p, p, q; mov.b64 {%0, %1}, p;}"
        : "+f"(x), "+f"(y)
        : "f"(a), "f"(b));
}

// Lane counts are accumulated in floats seeded with 2^23, so the float's bit
// pattern is 0x4B000000 + count; REDUX.SUM over 32 lanes then yields
// kCountBias + row count, compared directly against k + kCountBias.
constexpr unsigned kLaneBias = 0x4B000000u;
constexpr int kCountBias = (int)(32u * kLaneBias);  // 0x60000000 (mod 2^32)

__device__ __forceinline__ int warp_count(int lane_biased) {
    return (int)((unsigned)__reduce_add_sync(kFull, lane_biased));
}

// Midpoint when |a|, |b| < 2^126 (no overflow possible): RN((a+b)) * 0.5.
__device__ __forceinline__ float mid_fast(float a, float b) { return __fmul_rn(__fadd_rn(a, b), 0.5f); }

// General midpoint, bit-identical to F32((F64(a)+F64(b))*0.5) (Appendix C).
__device__ __forceinline__ float mid_exact(float a, float b) {
    float s = __fadd_rn(a, b);
    if (isinf(s) && isfinite(a) && isfinite(b)) return __fadd_rn(__fmul_rn(a, 0.5f), __fmul_rn(b, 0.5f));
    return __fmul_rn(s, 0.5f);
}

__device__ __forceinline__ float4 ld_stream4(const float* p) {
    return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float ld_stream1(const float* p) { return __ldcs(p); }


__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Asynchronous global -> shared copies (LDGSTS), 16 bytes each; src_bytes = 0
// zero-fills (padding groups).  Bypass L1 (.cg): each byte is read once.
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src, unsigned src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ float4 lds128(unsigned addr) {
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(addr) : "memory");
    return r;
}

// Shared-memory staging of selected (value, index) pairs: 8 bytes per output
// position, one buffer of k pairs per warp, addressed in the shared window.
__device__ __forceinline__ void stage_put(unsigned addr, float v, int idx) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(__float_as_int(v)), "r"(idx) : "memory");
}
__device__ __forceinline__ void stage_get(unsigned addr, float& v, int& idx) {
    int b;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(b), "=r"(idx) : "r"(addr) : "memory");
    v = __int_as_float(b);
}

// Inclusive warp prefix sum: SHFL.UP with its in-range predicate guarding the add.
__device__ __forceinline__ unsigned warp_incl_scan(unsigned x) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm volatile(
            "{.reg .pred p; .reg .b32 t;\n\t"
            "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
            "@p add.u32 %0, %0, t;}"
            : "+r"(x)
            : "r"(d));
    return x;
}

// ------------------------------------------------------- register row tile
//
// Slot (c, s) of lane l holds element c*32*V + l*V + s: chunk-major, so each
// 128-bit load of a warp covers 512 contiguous bytes, and index order is
// (chunk, lane, s) lexicographic -- a per-chunk lane scan gives positions.
// Padding slots (MASKED, last chunk only) hold NaN, which no >= test counts.
template <int V, int C, bool MASKED>
struct RegRow {
    static constexpr bool kStaged = true;  // selection goes through shared memory
    static constexpr bool kBlock = false;  // one warp per row
    static constexpr int kPad = 0;         // staging holds exactly k entries
    __host__ __device__ static constexpr unsigned stage_bytes(int k) { return (8u * (unsigned)k + 15u) & ~15u; }
    static constexpr int kV = V;
    static constexpr int kC = C;
    float v[C][V];

    __device__ __forceinline__ static int index(int c, int lane, int s) { return c * 32 * V + lane * V + s; }
    // V == 4 tiles are sized so only the last chunk can be partial; V == 1
    // tiles round C up to a power of two, so any chunk may be (partly) padding.
    __device__ __forceinline__ static bool valid(int c, int lane, int s, int m) {
        return !MASKED || (V == 4 && c < C - 1) || index(c, lane, s) < m;
    }

    __device__ __forceinline__ void load(const float* __restrict__ p, int m, int lane) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if constexpr (V == 4) {
                if (valid(c, lane, 0, m)) {
                    float4 q = ld_stream4(p + index(c, lane, 0));
                    v[c][0] = q.x; v[c][1] = q.y; v[c][2] = q.z; v[c][3] = q.w;
                } else {
                    v[c][0] = v[c][1] = v[c][2] = v[c][3] = __int_as_float(0x7fffffff);
                }
            } else {
#pragma unroll
                for (int s = 0; s < V; ++s)
                    v[c][s] = valid(c, lane, s, m) ? ld_stream1(p + index(c, lane, s)) : __int_as_float(0x7fffffff);
            }
        }
    }

    // Lane-local min (NaN-propagating, so a NaN anywhere in the row is seen)
    // and max (NaN-ignoring); padding is excluded.
    __device__ __forceinline__ void lane_min_max(int m, int lane, float& mn, float& mx) const {
        mn = __int_as_float(0x7f800000);
        mx = __int_as_float(0xff800000);
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
            for (int s = 0; s < V; ++s) {
                if (valid(c, lane, s, m)) mn = fmin_nan(mn, v[c][s]);
                mx = fmaxf(mx, v[c][s]);
            }
    }

    // Biased lane count of v >= t (see kLaneBias): FSET.BF + FADD2 per pair.
    __device__ __forceinline__ static int lane_valid(int, int) { return 0; }  // unused (no hint)

    __device__ __forceinline__ int lane_count_ge(float t) const {
        constexpr int kSlots = C * V;
        float sx = __int_as_float((int)kLaneBias), sy = 0.0f;
#pragma unroll
        for (int i = 0; i + 1 < kSlots; i += 2)
            add2(sx, sy, set_ge(v[i / V][i % V], t), set_ge(v[(i + 1) / V][(i + 1) % V], t));
        if constexpr (kSlots % 2) sx += set_ge(v[C - 1][V - 1], t);
        return __float_as_int(sx + sy);
    }

    // Per-chunk lane counts of the predicate bits packed one byte per chunk
    // (4 chunks per word: a lane holds <= 4 hits per chunk, a chunk <= 128),
    // so one warp scan serves four chunks.
    static constexpr int kWords = (C + 3) / 4;

    // Stage the first k elements (ascending index) with v >= t into the
    // warp's shared-memory row buffer (_kernels.py:118-125, 205-212).
    __device__ __forceinline__ unsigned select_ge(float t, int k, unsigned sbase, int lane, int) const {
        bool p[C][V];
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
            for (int s = 0; s < V; ++s) p[c][s] = v[c][s] >= t;
        if constexpr (V == 1) {
            const unsigned lt = lanemask_lt();
            int base = 0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (base >= k) break;
                const unsigned b = __ballot_sync(kFull, p[c][0]);
                const int pos = base + __popc(b & lt);
                if (p[c][0] && pos < k) stage_put(sbase + 8u * pos, v[c][0], index(c, lane, 0));
                base += __popc(b);
            }
        } else {
            unsigned cnt[kWords], incl[kWords], tot[kWords];
#pragma unroll
            for (int w = 0; w < kWords; ++w) cnt[w] = 0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                unsigned cl = 0;
#pragma unroll
                for (int s = 0; s < V; ++s) cl += p[c][s] ? 1u : 0u;
                cnt[c / 4] += cl << (8 * (c % 4));
            }
#pragma unroll
            for (int w = 0; w < kWords; ++w) {
                incl[w] = warp_incl_scan(cnt[w]);
                tot[w] = __shfl_sync(kFull, incl[w], 31);
            }
            int base = 0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int pos0 = base + (int)(((incl[c / 4] - cnt[c / 4]) >> (8 * (c % 4))) & 0xffu);
                unsigned addr = sbase + 8u * pos0;
                const unsigned aend = sbase + 8u * k;
#pragma unroll
                for (int s = 0; s < V; ++s) {
                    if (p[c][s] && addr < aend) stage_put(addr, v[c][s], index(c, lane, s));
                    addr += p[c][s] ? 8u : 0u;
                }
                base += (int)((tot[c / 4] >> (8 * (c % 4))) & 0xffu);
            }
        }
        return 0u;
    }

    // All elements >= t plus the first `need` elements of [lo, t), merged in
    // ascending index order (_kernels.py:126-145).  Cold on benchmark data.
    __device__ __forceinline__ void select_fill(float t, float lo, int need, int k, unsigned sbase,
                                                int lane) const {
        int baseA = 0, baseB = 0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            bool pa[V], pb[V];
            unsigned packed = 0;
#pragma unroll
            for (int s = 0; s < V; ++s) {
                pa[s] = v[c][s] >= t;
                pb[s] = (lo <= v[c][s]) && (v[c][s] < t);
                packed += (pa[s] ? 1u : 0u) + (pb[s] ? 0x10000u : 0u);
            }
            const unsigned incl = warp_incl_scan(packed);
            const unsigned total = __shfl_sync(kFull, incl, 31);
            const unsigned excl = incl - packed;
            int ea = baseA + (int)(excl & 0xffffu), eb = baseB + (int)(excl >> 16);
#pragma unroll
            for (int s = 0; s < V; ++s) {
                if (pa[s]) {
                    const int pos = ea + min(eb, need);
                    if (pos < k) stage_put(sbase + 8u * pos, v[c][s], index(c, lane, s));
                    ++ea;
                } else if (pb[s]) {
                    if (eb < need && ea + eb < k) stage_put(sbase + 8u * (ea + eb), v[c][s], index(c, lane, s));
                    ++eb;
                }
            }
            baseA += (int)(total & 0xffffu);
            baseB += (int)(total >> 16);
        }
    }
};

// Copy a staged row (k values, k indices in shared memory) to global with
// coalesced stores; the surrounding __syncwarp()s order the warp's shared
// buffer between rows.
__device__ __forceinline__ void flush_row(unsigned sbase, int k, float* __restrict__ ov, int* __restrict__ oi,
                                          int lane) {
    __syncwarp();
#pragma unroll 1
    for (int j = lane; j < k; j += 32) {
        float v;
        int i;
        stage_get(sbase + 8u * j, v, i);
        ov[j] = v;
        oi[j] = i;
    }
    __syncwarp();
}

// ------------------------------------------------- lane-contiguous row tile
//
// The register layout of the vectorised path: lane l holds the E consecutive
// elements [l*E, l*E + E) of the row (E a multiple of 4, E*32 >= M), loaded
// with 256-bit LDG.E.256 (WIDE: E % 8 == 0, unmasked, 32-byte aligned rows)
// or 128-bit loads.  Index order
// is (lane, slot), so one warp exclusive scan of the per-lane hit counts gives
// every selected element its output position.  Padding slots hold NaN.
template <int E, bool MASKED, bool WIDE = false>
struct LaneRow {
    static constexpr bool kStaged = true;
    static constexpr bool kBlock = false;
    static constexpr int kSlots = E;
    static constexpr int kPad = 32 * E;  // staging entries per warp
    float v[E];

    __device__ __forceinline__ static bool valid(int lane, int q, int m) { return !MASKED || lane * E + q < m; }

    __device__ __forceinline__ void load(const float* __restrict__ p, int m, int lane) {
        const float* lp = p + lane * E;
        if constexpr (WIDE && !MASKED && E % 8 == 0) {
#pragma unroll
            for (int g = 0; g < E / 8; ++g) {
                float* d = v + 8 * g;
                asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3]), "=f"(d[4]), "=f"(d[5]), "=f"(d[6]),
                               "=f"(d[7])
                             : "l"(lp + 8 * g));
            }
        } else {
#pragma unroll
            for (int g = 0; g < E / 4; ++g) {
                if (valid(lane, 4 * g, m)) {
                    const float4 q = ld_stream4(lp + 4 * g);
                    v[4 * g] = q.x; v[4 * g + 1] = q.y; v[4 * g + 2] = q.z; v[4 * g + 3] = q.w;
                } else {
                    v[4 * g] = v[4 * g + 1] = v[4 * g + 2] = v[4 * g + 3] = __int_as_float(0x7fffffff);
                }
            }
        }
    }

    // 16-bit rows (In = __nv_bfloat16 / __half), widened to fp32 exactly:
    // one 16-byte load per lane (WIDE: E = 8, unmasked, 16-byte aligned rows)
    // or 8-byte loads per 4 slots; padding slots hold NaN.
    template <class In>
    __device__ __forceinline__ void load16(const In* __restrict__ p, int m, int lane) {
        const In* lp = p + lane * E;
        unsigned w[E / 2];
        if constexpr (WIDE && !MASKED && E % 8 == 0) {
#pragma unroll
            for (int g = 0; g < E / 8; ++g)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(w[4 * g]), "=r"(w[4 * g + 1]), "=r"(w[4 * g + 2]), "=r"(w[4 * g + 3])
                             : "l"(lp + 8 * g));
        } else {
#pragma unroll
            for (int g = 0; g < E / 4; ++g) {
                if (valid(lane, 4 * g, m)) {
                    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                                 : "=r"(w[2 * g]), "=r"(w[2 * g + 1])
                                 : "l"(lp + 4 * g));
                } else {
                    w[2 * g] = w[2 * g + 1] = 0xffffffffu;  // NaN in both formats
                }
            }
        }
#pragma unroll
        for (int h = 0; h < E / 2; ++h) {
            if constexpr (std::is_same<In, __nv_bfloat16>::value) {
                v[2 * h] = __uint_as_float(w[h] << 16);
                v[2 * h + 1] = __uint_as_float(w[h] & 0xffff0000u);
            } else {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[h]));
                v[2 * h] = f.x;
                v[2 * h + 1] = f.y;
            }
        }
    }

    // Shared-memory image of a row (cp.async ring slots, the selection row
    // copy): lane l's E values at l * kLaneStride.  The stride is padded to an
    // odd number of 16-byte chunks, so the 8 lanes of each LDS.128/STS.128
    // phase hit 8 distinct bank groups (an unpadded 4E-byte stride is an
    // 8-way conflict at E = 32, 4-way at E = 16).
    static constexpr unsigned kChunks = E / 4;
    static constexpr unsigned kLaneStride = 16u * (kChunks | 1u);
    static constexpr unsigned kRowBytes = 32u * kLaneStride;
    // The warp copies a row in 512-byte coalesced pieces (lane l: bytes
    // [512 g + 16 l, +16) of the row) and sends each 16-byte chunk to its
    // owner lane's slot: element e = 128 g + 4 l lives in lane e / E, chunk
    // (e % E) / 4 (constant divisors; for E | 128 the offsets are
    // base + g * const).  Chunks past M are skipped (M % 4 == 0 here).
    __device__ __forceinline__ static unsigned slot_offset(int lane) { return (unsigned)lane * kLaneStride; }

    // salt: 0 at run time but opaque to the compiler (token & opaque_zero);
    // at E > 32 it keeps the per-chunk offsets and masks from being hoisted
    // out of the row loop, where kChunks of them would be held live (and
    // spill); narrower tiles keep the hoisted offsets (measured faster).
    static constexpr bool kSaltStage = E > 32;
    __device__ __forceinline__ static void stage_async(const float* __restrict__ p, int m, int lane, unsigned slot,
                                                       unsigned salt = 0u) {
        const float* src = p + 4 * lane;
        const unsigned e0 = 4u * (unsigned)lane + (kSaltStage ? salt : 0u);
#pragma unroll
        for (int g = 0; g < (int)kChunks; ++g) {
            const unsigned e = 128u * g + e0;
            const unsigned dst = slot + (e / E) * kLaneStride + 16u * ((e % E) / 4u);
            // chunks past M are not copied (load_smem masks those slots), so
            // every copy has the immediate size 16 and no per-chunk register
            if (!MASKED || (int)e < m) cp_async16(dst, src + 128 * g, 16u);
        }
    }

    __device__ __forceinline__ void load_smem(unsigned slot, int m, int lane) {
        const unsigned src = slot + slot_offset(lane);
        const int nv = m - lane * E;  // real slots of this lane (MASKED)
#pragma unroll
        for (int g = 0; g < E / 4; ++g) {
            const float4 q = lds128(src + 16u * g);
            const bool ok = !MASKED || 4 * g < nv;
            const float nan = __int_as_float(0x7fffffff);
            v[4 * g] = ok ? q.x : nan;
            v[4 * g + 1] = ok ? q.y : nan;
            v[4 * g + 2] = ok ? q.z : nan;
            v[4 * g + 3] = ok ? q.w : nan;
        }
    }

    // 16-bit rows in a ring slot (long-row kernel, rtk_rowtopk_x16): lane l's
    // E halves at l * kLaneStride16 (odd number of 16-byte chunks, as for
    // fp32); the row is copied in 512-byte coalesced pieces, each 16-byte
    // chunk (8 halves) sent to its owner lane.  Needs E % 8 == 0 and
    // M % 8 == 0 (whole chunks); chunks past M are not copied (NaN-prefilled:
    // a 0x7fff half is NaN in both formats).
    static constexpr unsigned kChunks16 = E / 8;
    static constexpr unsigned kLaneStride16 = 16u * (kChunks16 | 1u);
    static constexpr unsigned kRowBytes16 = 32u * kLaneStride16;
    template <class In>
    __device__ __forceinline__ static void stage_async16(const In* __restrict__ p, int m, int lane, unsigned slot,
                                                         unsigned salt = 0u) {
        static_assert(E % 8 == 0, "16-bit staging needs whole 16-byte chunks per lane");
        const In* src = p + 8 * lane;
        const unsigned e0 = 8u * (unsigned)lane + (kSaltStage ? salt : 0u);
#pragma unroll
        for (int g = 0; g < (int)kChunks16; ++g) {
            const unsigned e = 256u * g + e0;
            const unsigned dst = slot + (e / E) * kLaneStride16 + 16u * ((e % E) / 8u);
            if (!MASKED || (int)e < m) cp_async16(dst, src + 256 * g, 16u);
        }
    }
    template <class In>
    __device__ __forceinline__ void load_smem16(unsigned slot, int lane) {
        const unsigned src = slot + (unsigned)lane * kLaneStride16;
#pragma unroll
        for (int g = 0; g < E / 8; ++g) {
            const float4 q = lds128(src + 16u * g);
            const unsigned w[4] = {__float_as_uint(q.x), __float_as_uint(q.y), __float_as_uint(q.z),
                                   __float_as_uint(q.w)};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if constexpr (std::is_same<In, __nv_bfloat16>::value) {
                    v[8 * g + 2 * h] = __uint_as_float(w[h] << 16);
                    v[8 * g + 2 * h + 1] = __uint_as_float(w[h] & 0xffff0000u);
                } else {
                    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[h]));
                    v[8 * g + 2 * h] = f.x;
                    v[8 * g + 2 * h + 1] = f.y;
                }
            }
        }
    }

    // Unmasked read of a slot whose padding chunks hold NaN already (see
    // fill_slot_nan): no per-element select, so the LDS results are the tile.
    __device__ __forceinline__ void load_smem_prefilled(unsigned slot, int lane) {
        const unsigned src = slot + slot_offset(lane);
#pragma unroll
        for (int g = 0; g < E / 4; ++g) {
            const float4 q = lds128(src + 16u * g);
            v[4 * g] = q.x; v[4 * g + 1] = q.y; v[4 * g + 2] = q.z; v[4 * g + 3] = q.w;
        }
    }
    // NaN into every chunk of a slot (stage_async never writes the chunks past
    // M, so they stay NaN for every row of the launch).
    __device__ __forceinline__ static void fill_slot_nan(unsigned slot, int lane, unsigned bytes = kRowBytes) {
        const float nan = __int_as_float(0x7fffffff);
#pragma unroll 1
        for (unsigned i = (unsigned)lane; i < bytes / 16u; i += 32u)
            asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(slot + 16u * i), "f"(nan) : "memory");
    }

    __device__ __forceinline__ void lane_min_max(int m, int lane, float& mn, float& mx) const {
        mn = __int_as_float(0x7f800000);
        mx = __int_as_float(0xff800000);
        if constexpr (MASKED) {
            // padding slots (NaN) are a suffix of the lane's slots; fmin_nan
            // must not see them
            const int nv = m - lane * E;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                mn = fmin_nan(mn, q < nv ? v[q] : mn);
                mx = fmaxf(mx, v[q]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < E; ++q) {
                mn = fmin_nan(mn, v[q]);
                mx = fmaxf(mx, v[q]);
            }
        }
    }

    __device__ __forceinline__ int lane_count_ge(float t) const {
        float sx = set_ge(v[0], t), sy = set_ge(v[1], t);
#pragma unroll
        for (int q = 2; q < E; q += 2) add2(sx, sy, set_ge(v[q], t), set_ge(v[q + 1], t));
        return __float_as_int(__fadd_rn(__fadd_rn(sx, sy), 0x1p23f));  // kLaneBias + count
    }

    // Number of real (non-padding) slots of this lane.
    __device__ __forceinline__ static int lane_valid(int m, int lane) {
        return MASKED ? max(0, min(E, m - lane * E)) : E;
    }

    // Selection staging (per warp, kStageBytes of shared memory): a copy of
    // the row (padded layout, see kLaneStride) followed by the selected
    // indices in output order (32 E slots).  Only indices are staged per
    // element (one predicated STS.32 each, no register pairing); flush()
    // looks the values up in the row copy.
    static constexpr unsigned kIdxOff = kRowBytes;
    static constexpr unsigned kStageBytes = kRowBytes + 4u * 32u * E;
    __host__ __device__ static constexpr unsigned stage_bytes(int) { return kStageBytes; }

    // Shared-memory address of element i in the row copy at sbase.
    __device__ __forceinline__ static unsigned copy_addr(unsigned sbase, unsigned i) {
        return sbase + (i / E) * kLaneStride + 4u * (i % E);
    }

    // A staged index is always < 32*E for NaN-free rows (#{v >= t} >= k);
    // NaN rows (reported as an error) may leave slots unwritten, so clamp
    // before using an index as a shared-memory offset.
    __device__ __forceinline__ static unsigned clamp_slot(int i) {
        return ((32u * E) & (32u * E - 1)) == 0 ? (unsigned)i & (32u * E - 1) : min((unsigned)i, 32u * E - 1);
    }

    __device__ __forceinline__ void stage_row(unsigned sbase, int lane) const {
        const unsigned dst = sbase + slot_offset(lane);
#pragma unroll
        for (int g = 0; g < E / 4; ++g)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16u * g), "f"(v[4 * g]),
                         "f"(v[4 * g + 1]), "f"(v[4 * g + 2]), "f"(v[4 * g + 3])
                         : "memory");
    }

    // Stage this lane's elements with v >= t at output positions excl,
    // excl + 1, ... (excl: exclusive prefix of the lane hit counts).
    __device__ __forceinline__ void stage_idx(float t, unsigned sbase, int lane, unsigned excl) const {
        unsigned addr = sbase + kIdxOff + 4u * excl;
        const int i0 = lane * E;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            if (v[q] >= t) {
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(i0 + q) : "memory");
                addr += 4u;
            }
        }
    }

    // Stage every element with v >= t at its output position (the caller
    // guarantees #{v >= t} >= k and flushes only the first k entries; the
    // staging buffer holds 32*E entries, so no per-element cutoff is needed).
    // lane_hits: #{v >= t} in this lane, already known from the search pass
    // at t (the lane input of that pass's REDUX).
    __device__ __forceinline__ unsigned select_ge(float t, int, unsigned sbase, int lane, int lane_hits) const {
        stage_row(sbase, lane);
        const unsigned cl = (unsigned)lane_hits;
        const unsigned excl = warp_incl_scan(cl) - cl;
        stage_idx(t, sbase, lane, excl);
        return 0u;
    }

    // All v >= t plus the first `need` elements of [lo, t), ascending index
    // (_kernels.py:126-145).  Cold on benchmark data.
    __device__ __forceinline__ void select_fill(float t, float lo, int need, int, unsigned sbase, int lane) const {
        stage_row(sbase, lane);
        bool pa[E], pb[E];
        unsigned packed = 0;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            pa[q] = v[q] >= t;
            pb[q] = (lo <= v[q]) && (v[q] < t);
            packed += (pa[q] ? 1u : 0u) + (pb[q] ? 0x10000u : 0u);
        }
        const unsigned excl = warp_incl_scan(packed) - packed;
        int ea = (int)(excl & 0xffffu), eb = (int)(excl >> 16);
        const int i0 = lane * E;
        const unsigned ib = sbase + kIdxOff;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            if (pa[q]) {
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(ib + 4u * (ea + min(eb, need))), "r"(i0 + q) : "memory");
                ++ea;
            } else if (pb[q]) {
                if (eb < need) asm volatile("st.shared.b32 [%0], %1;" ::"r"(ib + 4u * (ea + eb)), "r"(i0 + q) : "memory");
                ++eb;
            }
        }
    }

    // Write the first k staged (value, index) pairs with coalesced stores.
    __device__ __forceinline__ static void flush(unsigned sbase, int k, float* __restrict__ ov, int* __restrict__ oi,
                                                 int lane) {
        __syncwarp();
#pragma unroll 1
        for (int j = lane; j < k; j += 32) {
            int i;
            float x;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(i) : "r"(sbase + kIdxOff + 4u * j) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(copy_addr(sbase, clamp_slot(i))) : "memory");
            ov[j] = x;
            oi[j] = i;
        }
        __syncwarp();
    }
};

// Lane-contiguous tile with cut-off selection staging: only lanes whose
// first hit falls among the first k output positions stage their hits, as
// (value, index) pairs; the lane straddling position k stages all of its
// hits into E pairs of slack, so no per-element cut-off test is needed
// (8(k + E) bytes per warp, the first k flushed by flush_row).  Long rows
// need little shared memory.  Used by the big-row kernel (rtk_big.cuh).
#ifndef RTK_CUT_SLACK
#define RTK_CUT_SLACK 1
#endif
template <int E, bool MASKED>
struct LaneRowCut : LaneRow<E, MASKED, false> {
    using Base = LaneRow<E, MASKED, false>;
    using Base::v;
    static constexpr int kPad = 0;  // flush_row writes the first k staged pairs
    __host__ __device__ static constexpr unsigned stage_bytes(int k) {
        return (8u * (unsigned)(k + (RTK_CUT_SLACK ? E : 0)) + 15u) & ~15u;
    }

    // Staging addresses are computed a group of G slots ahead of the stores
    // and all kept live until the group's stores have issued (folded into the
    // returned sink), so ptxas cannot recycle one address register for the
    // whole chain -- which would make every store wait for the previous
    // STS to read its operands (a serial WAR chain through the MIO queue).
    __device__ __forceinline__ unsigned select_ge(float t, int k, unsigned sbase, int lane, int lane_hits) const {
        constexpr int G = (E % 8 == 0) ? 8 : 4;
        const unsigned cl = (unsigned)lane_hits;
        const unsigned excl = warp_incl_scan(cl) - cl;
        unsigned addr = sbase + 8u * excl;
        const unsigned aend = sbase + 8u * (unsigned)k;
        const bool lane_on = excl < (unsigned)k;  // this lane's hits start before position k
        const int i0 = lane * E;
        unsigned sink = 0;
#pragma unroll
        for (int g = 0; g < E; g += G) {
            unsigned ad[G];
            bool p[G];
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const bool hit = v[g + q] >= t;
                p[q] = hit && (RTK_CUT_SLACK ? lane_on : addr < aend);
                ad[q] = addr;
                addr += hit ? 8u : 0u;
            }
#pragma unroll
            for (int q = 0; q < G; ++q)
                if (p[q]) stage_put(ad[q], v[g + q], i0 + g + q);
#pragma unroll
            for (int q = 0; q < G; ++q) sink ^= ad[q];
        }
        return sink;
    }

    // (cold; the compares are redone in the second pass rather than kept
    // as 2E predicates, which would raise the register bound of the kernel)
    __device__ __forceinline__ void select_fill(float t, float lo, int need, int k, unsigned sbase, int lane) const {
        unsigned packed = 0;
#pragma unroll
        for (int q = 0; q < E; ++q)
            packed += (v[q] >= t ? 1u : 0u) + ((lo <= v[q]) && (v[q] < t) ? 0x10000u : 0u);
        const unsigned excl = warp_incl_scan(packed) - packed;
        int ea = (int)(excl & 0xffffu), eb = (int)(excl >> 16);
        const int i0 = lane * E;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            if (v[q] >= t) {
                const int pos = ea + min(eb, need);
                if (pos < k) stage_put(sbase + 8u * pos, v[q], i0 + q);
                ++ea;
            } else if (lo <= v[q]) {
                if (eb < need && ea + eb < k) stage_put(sbase + 8u * (ea + eb), v[q], i0 + q);
                ++eb;
            }
        }
    }
};

// ------------------------------------------------------ global-memory row
//
// Rows longer than the register tile: same layout with V = 1 and a runtime
// chunk count, every pass re-reading the row (L1/L2 resident after pass 1).
struct GlobalRow {
    static constexpr bool kStaged = false;  // selection stores straight to global
    static constexpr bool kBlock = false;
    static constexpr int kPad = 0;
    __host__ __device__ static constexpr unsigned stage_bytes(int) { return 0u; }
    const float* __restrict__ p;
    int m;

    __device__ __forceinline__ void load(const float* __restrict__ ptr, int m_, int) {
        p = ptr;
        m = m_;
    }
    __device__ __forceinline__ float at(int e) const { return e < m ? __ldg(p + e) : __int_as_float(0x7fffffff); }

    __device__ __forceinline__ void lane_min_max(int, int lane, float& mn, float& mx) const {
        mn = __int_as_float(0x7f800000);
        mx = __int_as_float(0xff800000);
        for (int e = lane; e < m; e += 32) {
            float x = __ldg(p + e);
            mn = fmin_nan(mn, x);
            mx = fmaxf(mx, x);
        }
    }
    __device__ __forceinline__ static int lane_valid(int, int) { return 0; }  // unused (no hint)

    __device__ __forceinline__ int lane_count_ge(float t) const {
        int cnt = 0;
        for (int e = threadIdx.x & 31; e < m; e += 32) cnt += (__ldg(p + e) >= t) ? 1 : 0;
        return (int)kLaneBias + cnt;
    }
    __device__ __forceinline__ unsigned select_ge(float t, int k, float* __restrict__ ov, int* __restrict__ oi,
                                                  int lane, int) const {
        int base = 0;
        const unsigned lt = lanemask_lt();
        for (int c0 = 0; c0 < m && base < k; c0 += 32) {
            const int e = c0 + lane;
            const float x = at(e);
            const bool q = x >= t;
            const unsigned b = __ballot_sync(kFull, q);
            const int pos = base + __popc(b & lt);
            if (q && pos < k) {
                ov[pos] = x;
                oi[pos] = e;
            }
            base += __popc(b);
        }
        return 0u;
    }
    __device__ __forceinline__ void select_fill(float t, float lo, int need, int k, float* __restrict__ ov,
                                                int* __restrict__ oi, int lane) const {
        int baseA = 0, baseB = 0;
        const unsigned lt = lanemask_lt();
        for (int c0 = 0; c0 < m; c0 += 32) {
            const int e = c0 + lane;
            const float x = at(e);
            const bool qa = x >= t;
            const bool qb = (lo <= x) && (x < t);
            const unsigned ba = __ballot_sync(kFull, qa), bb = __ballot_sync(kFull, qb);
            const int ea = baseA + __popc(ba & lt), eb = baseB + __popc(bb & lt);
            if (qa) {
                const int pos = ea + min(eb, need);
                if (pos < k) {
                    ov[pos] = x;
                    oi[pos] = e;
                }
            } else if (qb && eb < need) {
                const int pos = ea + eb;
                if (pos < k) {
                    ov[pos] = x;
                    oi[pos] = e;
                }
            }
            baseA += __popc(ba);
            baseB += __popc(bb);
        }
    }
};

// ---------------------------------------------------------- the searches

// Row-level reductions: one warp per row (warp collectives) or a CTA per
// row (Row::kBlock, rtk_block.cuh: warp collectives + a shared-memory
// combine; every thread of the CTA gets the row's value).
template <class Row>
__device__ __forceinline__ int row_count(const Row& row, int lane_biased) {
    if constexpr (Row::kBlock)
        return row.count(lane_biased);
    else
        return warp_count(lane_biased);
}
template <class Row>
__device__ __forceinline__ bool row_leader(int lane) {
    if constexpr (Row::kBlock)
        return threadIdx.x == 0;
    else
        return lane == 0;
}

// Algorithm 1 loop (_kernels.py:64-84), entered only when the loop-head test
// passed at it == 0.  FP: eps_rel == 0 and mx0 finite, so the float64 head
// test `mx - mn > eps` is the fp32 `mx > mn`; it is evaluated at the end of
// each body (before the next body's hard-cap test, the reference order).
// SAFE: |mn0|,|mx0| < 2^126 so the midpoint cannot overflow.
// cnt is returned biased by kCountBias.
template <bool FP, bool SAFE, class Row>
__device__ __forceinline__ int exact_loop(const Row& row, int kb, double eps, int cap, float& mn, float& mx,
                                          float& thres, int& cnt, int& it, int& lane_last) {
    float mid;
    if constexpr (FP && SAFE) {
        // mid = RN((mn+mx)/2) always lies in [mn, mx].  If it is strictly
        // inside, neither no-progress exit can fire and the updated bracket
        // still satisfies mx > mn; if it equals an endpoint the reference
        // exits after this body with INTERVAL_BELOW_EPSILON (stuck, or the
        // bracket collapses and the next head test fails) unless cnt == k.
        bool eq, inside;
        do {
            ++it;
            mid = mid_fast(mn, mx);
            inside = (mn < mid) && (mid < mx);
            lane_last = row.lane_count_ge(mid);
            cnt = row_count(row, lane_last);
            const bool lt = cnt < kb;
            eq = cnt == kb;
            mx = lt ? mid : mx;
            mn = lt ? mn : mid;
        } while (!eq && inside && it < cap);
        thres = mid;
        if (eq) return kExitCountEqualsK;
        return inside ? kExitHardCapReached : kExitIntervalBelowEps;
    } else {
        // General form: explicit no-progress tests and the float64 head test
        // (_kernels.py:65,78,82).  The bracket update is applied
        // unconditionally: on a no-progress exit it is a no-op.
        bool eq, stuck, cont;
        do {
            ++it;
            mid = SAFE ? mid_fast(mn, mx) : mid_exact(mn, mx);
            lane_last = row.lane_count_ge(mid);
            cnt = row_count(row, lane_last);
            const bool lt = cnt < kb;
            eq = cnt == kb;
            stuck = mid == (lt ? mx : mn);
            mx = lt ? mid : mx;
            mn = lt ? mn : mid;
            cont = FP ? (mx > mn) : ((double)mx - (double)mn > eps);
        } while (!eq && !stuck && cont && it < cap);
        thres = mid;
        if (eq) return kExitCountEqualsK;
        if (stuck || !cont) return kExitIntervalBelowEps;
        return kExitHardCapReached;
    }
}

// Fast form of the FP && SAFE loop for launches without traces: up to
// `steps` reference bisection steps with no no-progress tests, leaving the
// loop on cnt == k.  Why it is exact:
//   * mid = RN((mn+mx)/2) is strictly inside (mn, mx) whenever a float lies
//     strictly between them; otherwise it equals an endpoint ("stuck"), the
//     update below is then a no-op, and every later step repeats it.
//   * Before the first step with cnt == k, the bracket keeps
//     mn <= x_{k+1} < x_k <= mx (x_j = j-th largest); x_k is a float strictly
//     above mn, so a stuck step before the first cnt == k step means no
//     later step can ever reach cnt == k.  Hence when this loop leaves on
//     cnt == k, no reference exit fired earlier and the state equals the
//     reference's (COUNT_EQUALS_K at the same step).
//   * Otherwise the state after `steps` steps is the reference state (frozen
//     since the stuck step, if any); the caller resumes with exact_loop, whose
//     first step then reproduces the reference's INTERVAL_BELOW_EPSILON exit
//     (same mid, same count), or continues the search.  Only the reported
//     iteration of such a stuck exit would differ, and this form is not used
//     when traces are requested.
// Returns true on cnt == k; cnt biased by kCountBias.
template <class Row>
__device__ __forceinline__ bool exact_loop_fast(const Row& row, int kb, int steps, float& mn, float& mx, float& thres,
                                                int& cnt, int& it, int& lane_last) {
    float mid;
    int c, lc;
#pragma unroll 1
    for (;;) {
        ++it;
        mid = mid_fast(mn, mx);
        lc = row.lane_count_ge(mid);
        c = row_count(row, lc);
        const bool lt = c < kb;
        mx = lt ? mid : mx;
        mn = lt ? mn : mid;
        if (c == kb || it >= steps) break;
    }
    thres = mid;
    cnt = c;
    lane_last = lc;
    return c == kb;
}

#ifndef RTK_FAST_STEPS
#define RTK_FAST_STEPS 24  // fast steps before the general loop takes over (stuck rows)
#endif

// Algorithm 2 loop (_kernels.py:96-102): exactly max_iter steps; also tracks
// this lane's count at the final lower bound (the selection threshold).
template <bool SAFE, class Row>
__device__ __forceinline__ void early_loop(const Row& row, int kb, int max_iter, float& mn, float& mx, int& lane_mn) {
    for (int i = 0; i < max_iter; ++i) {
        const float mid = SAFE ? mid_fast(mn, mx) : mid_exact(mn, mx);
        const int lc = row.lane_count_ge(mid);
        const bool lt = row_count(row, lc) < kb;
        mx = lt ? mid : mx;
        mn = lt ? mn : mid;
        lane_mn = lt ? lane_mn : lc;
    }
}

// Staged rows: LaneRow stages indices + a row copy (LaneRow::flush), RegRow
// stages (value, index) pairs (flush_row).
// dep: the staging sink ANDed with opaque_zero (0 at run time); adding it
// to the flush addresses keeps the staging addresses live (LaneRowCut).
template <class Row>
__device__ __forceinline__ void flush_staged(unsigned sbase, int k, float* __restrict__ ov, int* __restrict__ oi,
                                             int lane, unsigned dep = 0u) {
    if constexpr (Row::kBlock)
        Row::flush_block(sbase + dep, k, ov, oi);
    else if constexpr (Row::kPad > 0)
        Row::flush(sbase + dep, k, ov, oi, lane);
    else
        flush_row(sbase + dep, k, ov, oi, lane);
}

struct NoHook {
    __device__ __forceinline__ void operator()(unsigned) const {}
};

// Byte offset of row r in a matrix with row stride `ld_bytes` (< 2^32).
template <class T>
__device__ __forceinline__ T* row_ptr(T* base, unsigned r, unsigned ld_bytes) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + (unsigned long long)r * ld_bytes);
}
template <class T>
__device__ __forceinline__ const T* row_ptr(const T* base, unsigned r, unsigned ld_bytes) {
    return reinterpret_cast<const T*>(reinterpret_cast<const char*>(base) + (unsigned long long)r * ld_bytes);
}

// select_exact (_kernels.py:149-162): threshold t = mx when the search
// ended with cnt > k (eps_rel == 0, not degenerate), else thres; then
// select_threshold (_kernels.py:106-146) with lo = mn.  cnt is biased.
template <class Row>
__device__ __forceinline__ void select_exact(const Row& row, const Args& a, int lane, unsigned sbase, bool fp,
                                             int reason, float thres, float mn, float mx, int cnt, int lane_t,
                                             float* __restrict__ ov, int* __restrict__ oi) {
    const int k = a.k;
    const bool use_mx = (cnt > k + kCountBias) && fp && (reason != kExitDegenerateRow);
    float t = thres;
    int ca = cnt - kCountBias;
    if (use_mx) {
        t = mx;
        lane_t = row.lane_count_ge(mx);
        ca = row_count(row, lane_t) - kCountBias;
    }
    if constexpr (Row::kStaged) {
        unsigned sink = 0;
        if (ca >= k)
            sink = row.select_ge(t, k, sbase, lane, lane_t - (int)kLaneBias);
        else
            row.select_fill(t, mn, k - ca, k, sbase, lane);
        flush_staged<Row>(sbase, k, ov, oi, lane, sink & a.opaque_zero);
    } else {
        if (ca >= k)
            row.select_ge(t, k, ov, oi, lane, 0);
        else
            row.select_fill(t, mn, k - ca, k, ov, oi, lane);
    }
}

// Rows holding a NaN: record the first offending row (batch.py:37-39).  Cold.
static __device__ __noinline__ void report_nan(unsigned* nan_row, unsigned r, int lane) {
    if (lane == 0 && nan_row) atomicMin(nan_row, r);
}

// Everything after the row's min/max (mn0, mx0): search, selection, flush,
// traces -- the general per-row path (all modes, every exit rule).
template <int MODE, bool TRACES, class Row>
__device__ __forceinline__ void row_body(const Row& row, unsigned r, const Args& a, int lane, unsigned sbase, bool fp,
                                         float mn0, float mx0) {
    const int k = a.k;
    const int kb = k + kCountBias;
    const unsigned ldo_b = (unsigned)a.ldo * 4u;
    float* ov = row_ptr(a.vals, r, ldo_b);
    int* oi = row_ptr(a.idx, r, ldo_b);
    int it = 0, reason;
    const bool safe = fabsf(mn0) < 0x1p126f && fabsf(mx0) < 0x1p126f;

    if constexpr (MODE == kEarly) {
        // Algorithm 2 (_kernels.py:87-103) + first-k selection (:205-212)
        float mn = mn0, mx = mx0;
        int lane_mn = (int)kLaneBias + Row::lane_valid(a.m, lane);  // every element is >= mn0
        if (!(mx0 > mn0)) {
            reason = kExitDegenerateRow;
        } else {
            if (safe)
                early_loop<true>(row, kb, a.max_iter, mn, mx, lane_mn);
            else
                early_loop<false>(row, kb, a.max_iter, mn, mx, lane_mn);
            it = a.max_iter;
            reason = kExitMaxIterReached;
        }
        if constexpr (Row::kStaged) {
            const unsigned sink = row.select_ge(mn, k, sbase, lane, lane_mn - (int)kLaneBias);
            flush_staged<Row>(sbase, k, ov, oi, lane, sink & a.opaque_zero);
        } else {
            row.select_ge(mn, k, ov, oi, lane, 0);
        }
    } else {
        // Algorithm 1 (_kernels.py:48-84) + select_exact (_kernels.py:149-162);
        // fp: eps_rel == 0 (hoisted by the caller).
        float mn = mn0, mx = mx0, thres = mn0;
        int cnt = a.m + kCountBias;
        int lane_t = (int)kLaneBias + Row::lane_valid(a.m, lane);  // lane count at thres
        const int cap = a.hard_cap;
        if (fp) {
            if (!(isfinite(mx0) && mx0 > mn0)) {
                reason = kExitDegenerateRow;  // eps = 0*mx0 is NaN for infinite mx0
            } else if (safe) {
                if constexpr (!TRACES) {
                    const int steps = min(cap, RTK_FAST_STEPS);
                    if (exact_loop_fast(row, kb, steps, mn, mx, thres, cnt, it, lane_t))
                        reason = kExitCountEqualsK;
                    else if (it >= cap)
                        reason = kExitHardCapReached;  // selection below treats HARD_CAP and IBE alike
                    else
                        reason = exact_loop<true, true>(row, kb, 0.0, cap, mn, mx, thres, cnt, it, lane_t);
                } else {
                    reason = exact_loop<true, true>(row, kb, 0.0, cap, mn, mx, thres, cnt, it, lane_t);
                }
            } else {
                reason = exact_loop<true, false>(row, kb, 0.0, cap, mn, mx, thres, cnt, it, lane_t);
            }
        } else {
            const double eps = a.eps_rel * (double)mx0;
            if (!((double)mx0 - (double)mn0 > eps))
                reason = kExitDegenerateRow;
            else
                reason = exact_loop<false, false>(row, kb, eps, cap, mn, mx, thres, cnt, it, lane_t);
        }
        if constexpr (MODE == kExact) select_exact(row, a, lane, sbase, fp, reason, thres, mn, mx, cnt, lane_t, ov, oi);
    }
    if constexpr (TRACES) {
        if (row_leader<Row>(lane)) {
            a.iters[r] = it;
            a.reasons[r] = (signed char)reason;
        }
    }
}

// `after_load(token)` runs once the row's registers have been consumed by
// the lane-local min/max; `token` is derived from that min/max, so a load
// issued there with `token & opaque_zero` in its address cannot be hoisted
// above the consumption of this row (the next row's prefetch goes there).
template <int MODE, bool TRACES, class Row, class Hook = NoHook>
__device__ __forceinline__ void process_row(const Row& row, unsigned r, const Args& a, int lane, unsigned sbase,
                                            bool fp, const Hook& after_load = Hook()) {
    float mnl, mxl;
    row.lane_min_max(a.m, lane, mnl, mxl);
    after_load(__float_as_uint(mnl) ^ __float_as_uint(mxl));
    float mn0, mx0;
    if constexpr (Row::kBlock) {
        row.reduce_min_max(mnl, mxl, mn0, mx0);
    } else {
        mn0 = warp_min_nan(mnl);
        mx0 = warp_max(mxl);
    }
    // keep the (noinline) call warp-uniform: a divergent call site makes ptxas
    // guard every later collective with WARPSYNC / ENDCOLLECTIVE
    if (mn0 != mn0) report_nan(a.nan_row, r, row_leader<Row>(lane) ? 0 : 1);
    row_body<MODE, TRACES>(row, r, a, lane, sbase, fp, mn0, mx0);
}

// Persistent grid-stride row loop.  Each warp prefetches its next row into a
// second register tile once the current tile has been read by the lane
// min/max: the prefetch address carries `token & opaque_zero`, so ptxas
// cannot issue it earlier.  (Issued earlier, the two tiles' loads share one
// scoreboard slot and the first use of the current tile waits for the
// just-issued prefetch too -- a full DRAM latency per row.)  Past the last
// row the prefetch re-reads the last row.  Dynamic shared memory: one
// staging buffer of (value, index) pairs per warp (staged rows only).
// Row indices are 32-bit (the host checks n < 2^32 - 1, row strides < 2^30).
template <int MODE, class Row, bool TRACES>
__global__ void __launch_bounds__(RTK_CTA_THREADS, RTK_MIN_CTAS) rowtopk_kernel(Args a) {
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const unsigned per_warp = MODE == kTrace ? 0u : Row::stage_bytes(a.k);  // staging bytes
    // The warp index is broadcast from lane 0 so ptxas can prove every row
    // loop below warp-uniform (no BRA.DIV convergence checks before the
    // REDUX/SHFL collectives, and uniform registers for the row bookkeeping).
    const int wid = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem) + (unsigned)wid * per_warp;
    const unsigned wpc = blockDim.x >> 5;
    const unsigned nw = gridDim.x * wpc;
    const unsigned n = (unsigned)a.n;
    unsigned r = blockIdx.x * wpc + (unsigned)wid;
    if (r >= n) return;
    const unsigned lim = n > nw ? n - nw : 0u;  // rows below lim have a successor
    const unsigned ldx_b = (unsigned)a.ldx * 4u;
    const unsigned oz = a.opaque_zero;
    const bool fp = a.eps_rel == 0.0;
    Row A, B;
    A.load(row_ptr(a.x, r, ldx_b), a.m, lane);
    for (;;) {
        const bool more1 = r < lim;
        const unsigned r1 = more1 ? r + nw : r;
        process_row<MODE, TRACES>(A, r, a, lane, sbase, fp,
                                  [&](unsigned tok) { B.load(row_ptr(a.x, r1 + (tok & oz), ldx_b), a.m, lane); });
        if (!more1) break;
        r = r1;
        const bool more2 = r < lim;
        const unsigned r2 = more2 ? r + nw : r;
        process_row<MODE, TRACES>(B, r, a, lane, sbase, fp,
                                  [&](unsigned tok) { A.load(row_ptr(a.x, r2 + (tok & oz), ldx_b), a.m, lane); });
        if (!more2) break;
        r = r2;
    }
}

#ifdef RTK_DEFINE_FLAT_KERNELS  // defined once, in rtk_capi.cu
// k == M shortcut (_kernels.py:173-179): copy the row, indices 0..M-1, trace (0, DEGENERATE).
__global__ void __launch_bounds__(256) full_copy_kernel(Args a) {
    const long long total = a.n * (long long)a.m;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const long long r = e / a.m;
        const int j = (int)(e - r * a.m);
        const float x = a.x[r * a.ldx + j];
        if (a.vals) {
            a.vals[r * a.ldo + j] = x;
            a.idx[r * a.ldo + j] = j;
        }
        if (x != x && a.nan_row) atomicMin(a.nan_row, (unsigned)r);
        if (j == 0) {
            if (a.iters) a.iters[r] = 0;
            if (a.reasons) a.reasons[r] = (signed char)kExitDegenerateRow;
        }
    }
}

// k == M with 16-byte aligned rows (M, ldx, ldo multiples of 4): one float4
// of values and one int4 of indices per item, 32-bit row arithmetic
// (the host guarantees n * M / 4 < 2^32), streaming loads and stores.
__device__ __forceinline__ void copy_item4(const Args& a, unsigned r, unsigned c, float4 x) {
    const unsigned long long o = (unsigned long long)r * a.ldo + c;
    if (a.vals) {
        __stcs(reinterpret_cast<float4*>(a.vals + o), x);
        __stcs(reinterpret_cast<int4*>(a.idx + o), make_int4((int)c, (int)c + 1, (int)c + 2, (int)c + 3));
    }
    if ((x.x != x.x || x.y != x.y || x.z != x.z || x.w != x.w) && a.nan_row) atomicMin(a.nan_row, r);
    if (c == 0u) {
        if (a.iters) a.iters[r] = 0;
        if (a.reasons) a.reasons[r] = (signed char)kExitDegenerateRow;
    }
}

__global__ void __launch_bounds__(256) full_copy_vec4_kernel(Args a) {
    const unsigned m4 = (unsigned)a.m >> 2;
    const unsigned total = (unsigned)a.n * m4;
    const unsigned stride = gridDim.x * blockDim.x;
    // two items per thread and iteration, both loads issued before the stores
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += 2u * stride) {
        const unsigned e2 = e + stride;
        const unsigned r = e / m4, c = 4u * (e - r * m4);
        const unsigned r2 = e2 / m4, c2 = 4u * (e2 - r2 * m4);
        const float4 x = __ldcs(reinterpret_cast<const float4*>(a.x + (unsigned long long)r * a.ldx + c));
        float4 x2 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e2 < total) x2 = __ldcs(reinterpret_cast<const float4*>(a.x + (unsigned long long)r2 * a.ldx + c2));
        copy_item4(a, r, c, x);
        if (e2 < total) copy_item4(a, r2, c2, x2);
    }
}

// NaN scan (batch.py:37-39) as a standalone pass.
__global__ void __launch_bounds__(256) nan_scan_kernel(Args a) {
    const long long total = a.n * (long long)a.m;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const long long r = e / a.m;
        const int j = (int)(e - r * a.m);
        const float x = a.x[r * a.ldx + j];
        if (x != x) atomicMin(a.nan_row, (unsigned)r);
    }
}

// Per-row min/max (_kernels.py:26-36) and count (_kernels.py:39-45), warp per row.
__global__ void __launch_bounds__(256) min_max_kernel(Args a, float* __restrict__ mins, float* __restrict__ maxs) {
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.n; r += nw) {
        GlobalRow row;
        row.load(a.x + r * a.ldx, a.m, lane);
        float mn, mx;
        row.lane_min_max(a.m, lane, mn, mx);
        mn = warp_min_nan(mn);
        mx = warp_max(mx);
        if (lane == 0) {
            mins[r] = mn;
            maxs[r] = mx;
        }
    }
}

__global__ void __launch_bounds__(256) count_ge_kernel(Args a, const float* __restrict__ thres,
                                                       int* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.n; r += nw) {
        GlobalRow row;
        row.load(a.x + r * a.ldx, a.m, lane);
        const int c = warp_count(row.lane_count_ge(thres[r])) - kCountBias;
        if (lane == 0) counts[r] = c;
    }
}

#endif  // RTK_DEFINE_FLAT_KERNELS

}  // namespace rtk
