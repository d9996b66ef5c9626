/*
 * rtk.h -- C ABI of the B200-native row-wise top-k library (librtk.so).
 *
 * Drop-in boundary for the reference's operator layer
 *   /root/reference/pkg/src/rowtopk/_kernels.py
 * whose chunk kernels the reference batch engine calls per row chunk
 * (batch.py:125-128 and batch.py:133-136).  Conventions mirror that operator:
 *   - the caller allocates every output (batch.py:114-117); the library never
 *     allocates, frees or synchronises;
 *   - the caller validates arguments first (batch.py:107-112); the library
 *     re-checks sizes and returns RTK_EINVAL instead of raising;
 *   - calls are reentrant; concurrent calls must write disjoint outputs
 *     (batch.py:3-5).
 * Differences forced by the device boundary:
 *   - all array pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *     storage), work is enqueued asynchronously on `stream` (a cudaStream_t,
 *     NULL = legacy default stream);
 *   - NaN rejection (batch.py:37-39) is fused into the kernels: when
 *     `nan_first_row` is non-NULL it must point to one device uint32; the call
 *     resets it to 0xFFFFFFFF and the kernels atomically lower it to the index
 *     of the first row holding a NaN.  The caller reads it after the stream
 *     completes and raises NaNInputError (rows with NaN get unspecified output).
 *
 * Row layout: x is row-major, row r starts at x + r*ldx (m <= ldx < 2^30).
 * Outputs row r start at vals + r*ldo / idx + r*ldo (k <= ldo < 2^30); n < 2^32 - 1.  Exactly k values and
 * k int32 indices are written per row, indices ascending, values bit copies
 * of x (_kernels.py:106-146).  iters (int32) / reasons (int8, ExitReason codes
 * 1..5, _kernels.py:19-23) are per-row traces; both NULL turns trace
 * collection off (BatchConfig.collect_traces=False, batch.py:58), exactly one
 * NULL is RTK_EINVAL.
 *
 * Return value: RTK_OK, RTK_EINVAL (bad sizes, k not in [1, m], NULL
 * required pointer), or RTK_ECUDA (launch failure); rtk_last_error() then
 * returns a thread-local message.
 */
#ifndef RTK_H_
#define RTK_H_

#include <stdint.h>

#if defined(__GNUC__)
#define RTK_API __attribute__((visibility("default")))
#else
#define RTK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RTK_OK 0
#define RTK_EINVAL 1
#define RTK_ECUDA 2
#define RTK_EIO 3     /* file open/read/write failed (rtk_topk_file_f32) */
#define RTK_EFORMAT 4 /* bad magic or unsupported format version */
#define RTK_ETRUNC 5  /* file shorter than its header declares, or empty payload */
#define RTK_ENAN 6    /* the matrix holds a NaN (first offending row reported) */
#define RTK_EUNSUPPORTED 7 /* rtk_rowtopk_x16: shape/layout outside its native path */

#define RTK_EXIT_COUNT_EQUALS_K 1
#define RTK_EXIT_INTERVAL_BELOW_EPSILON 2
#define RTK_EXIT_MAX_ITER_REACHED 3
#define RTK_EXIT_HARD_CAP_REACHED 4
#define RTK_EXIT_DEGENERATE_ROW 5

/* Exact mode (Algorithm 1 + select_exact).  Replaces
 *   _kernels.exact_topk_chunk(data, k, eps_rel, hard_cap,
 *                             out_vals, out_idx, out_iters, out_reasons)
 *   (/root/reference/pkg/src/rowtopk/_kernels.py:165-186)
 * eps_rel >= 0 (SearchConfig.epsilon_rel), hard_cap >= 1 (select.py:36). */
RTK_API int rtk_rowtopk_exact_f32(const float *x, int64_t n, int64_t m, int64_t ldx, int32_t k,
                          double eps_rel, int32_t hard_cap, float *vals, int32_t *idx,
                          int64_t ldo, int32_t *iters, int8_t *reasons,
                          uint32_t *nan_first_row, void *stream);

/* Early-stop mode (Algorithm 2 + first-k selection).  Replaces
 *   _kernels.early_topk_chunk(data, k, max_iter,
 *                             out_vals, out_idx, out_iters, out_reasons)
 *   (/root/reference/pkg/src/rowtopk/_kernels.py:189-214)
 * max_iter >= 1 (SearchConfig.max_iter, select.py:37). */
RTK_API int rtk_rowtopk_early_f32(const float *x, int64_t n, int64_t m, int64_t ldx, int32_t k,
                          int32_t max_iter, float *vals, int32_t *idx, int64_t ldo,
                          int32_t *iters, int8_t *reasons, uint32_t *nan_first_row,
                          void *stream);

/* Row top-k of a 16-bit float matrix read natively (dtype 1 = bfloat16,
 * 2 = float16) and widened to float32 in registers.  The widening is exact,
 * so the outputs (float32 values, int32 indices) equal rtk_rowtopk_*_f32 on
 * the float32 image of x -- which is what the reference computes, since
 * as_matrix converts every input to float32 (batch.py:30-36) -- with half
 * the input bytes and no conversion pass.  mode 0 = exact (eps_rel = 0,
 * hard_cap), 1 = early stop (max_iter); no traces.  Native path: 1 <= k < m
 * and either m <= 256, m % 4 == 0, ldx % 4 == 0, x 8-byte aligned, or
 * 256 < m <= 4096, m % 8 == 0, ldx % 8 == 0, x 16-byte aligned; anything
 * else returns RTK_EUNSUPPORTED (convert to float32 and use the _f32 calls). */
RTK_API int rtk_rowtopk_x16(const void *x, int32_t dtype, int32_t mode, int64_t n, int64_t m, int64_t ldx,
                    int32_t k, int32_t hard_cap, int32_t max_iter, float *vals, int32_t *idx,
                    int64_t ldo, uint32_t *nan_first_row, void *stream);

/* Fused MaxK nonlinearity (MaxK-GNN): the row top-k of
 * rtk_rowtopk_*_f32 / rtk_rowtopk_x16 (same vals / idx outputs) and, from the
 * same kernel,
 *   - dense (nullable): the dense MaxK rows, dense + r*ldd holding row r of x
 *     with all but the k selected entries set to +0, in x's type (dtype 0 =
 *     float32, 1 = bfloat16, 2 = float16; selected entries are bit copies);
 *     replaces the select -> rtk_scatter_rows_f32 pair;
 *   - idx8 (nullable): the indices again as uint8 (m <= 256), row r at
 *     idx8 + r*ld8 (ld8 >= k): the compact index layout of the MaxK sparse
 *     rows consumed by rtk_maxk_spmm_f32.
 * At least one of dense / idx8 is non-NULL.  mode 0 = exact (eps_rel = 0,
 * hard_cap), 1 = early stop (max_iter); no traces.  Native path: m = 128 or
 * 256, 1 <= k < m, ldx a multiple of 4 with x 16-byte (float32) / 8-byte
 * (16-bit) aligned, dense rows 16-byte aligned (8-byte for 16-bit rows of
 * 128); anything else returns RTK_EUNSUPPORTED (use the unfused pair). */
RTK_API int rtk_maxk_dense(const void *x, int32_t dtype, int32_t mode, int64_t n, int64_t m, int64_t ldx,
                   int32_t k, int32_t hard_cap, int32_t max_iter, float *vals, int32_t *idx, int64_t ldo,
                   void *dense, int64_t ldd, uint8_t *idx8, int64_t ld8, uint32_t *nan_first_row,
                   void *stream);

/* Exit statistics only, no selection.  Replaces
 *   _kernels.exact_trace_chunk(data, k, eps_rel, hard_cap, out_iters, out_reasons)
 *   (/root/reference/pkg/src/rowtopk/_kernels.py:217-231)
 * iters and reasons are required here. */
RTK_API int rtk_exact_trace_f32(const float *x, int64_t n, int64_t m, int64_t ldx, int32_t k,
                        double eps_rel, int32_t hard_cap, int32_t *iters, int8_t *reasons,
                        uint32_t *nan_first_row, void *stream);

/* NaN scan only: the as_matrix validation pass (batch.py:37-39), used when
 * the caller must report NaN before a k-range error (batch.py:107-111). */
RTK_API int rtk_nan_scan_f32(const float *x, int64_t n, int64_t m, int64_t ldx, uint32_t *nan_first_row,
                     void *stream);

/* Per-row min/max (_kernels.row_min_max, _kernels.py:26-36) and inclusive
 * count (_kernels.count_ge, _kernels.py:39-45) as batched device ops, backing
 * the single-row helpers select.min_max / select.count_ge (select.py:116-129).
 * thres has one float per row; counts are int32. */
RTK_API int rtk_row_min_max_f32(const float *x, int64_t n, int64_t m, int64_t ldx, float *mins,
                        float *maxs, void *stream);
RTK_API int rtk_count_ge_f32(const float *x, int64_t n, int64_t m, int64_t ldx, const float *thres,
                     int32_t *counts, void *stream);

/* MaxK-GNN consumer shapes.  The row top-k output (values,
 * ascending int32 indices, k per row) is the fixed-k-per-row sparse layout
 * the MaxK-GNN aggregation consumes; these convert between it and dense rows.
 * rtk_scatter_rows_f32: out[r, idx[r,j]] = vals[r,j], 0 elsewhere (out is
 *   n x m with row stride ldo >= m; vals/idx share row stride ldv >= k);
 *   the MaxK nonlinearity's dense output, and the backward of the gather.
 * rtk_gather_rows_f32: vals[r,j] = dense[r, idx[r,j]] (dense row stride
 *   ldd >= m); the backward of the MaxK nonlinearity.
 * Indices outside [0, m) are skipped (scatter) / read as 0 (gather). */
RTK_API int rtk_scatter_rows_f32(const float *vals, const int32_t *idx, int64_t ldv, int64_t n, int32_t k,
                         int64_t m, float *out, int64_t ldo, void *stream);
RTK_API int rtk_gather_rows_f32(const float *dense, int64_t ldd, const int32_t *idx, int64_t ldv, int64_t n,
                        int32_t k, int64_t m, float *vals, void *stream);

/* MaxK-GNN aggregation over the fixed-k rows (the consumer of the row top-k
 * output): with the graph as CSR (row_ptr[n+1] int64, col int32,
 * aval f32 edge weights, NULL = all 1) and H the fixed-k matrix (row j: vals
 * at columns idx, k per row, row stride ldv; idx int32 or idx8 uint8 for
 * m <= 256 -- exactly one non-NULL),
 *   rtk_maxk_spmm_f32:          out[i, :] = sum_{e=(i,j)} aval[e] * H[j, :]
 *                               (out n x m, row stride ldo; m <= 1024);
 *   rtk_maxk_spmm_backward_f32: grad_vals[j, t] = sum_{e=(i,j)} aval[e] *
 *                               grad_out[i, idx[j, t]], over the TRANSPOSED
 *                               graph's CSR (row j lists the i with e=(i,j)).
 * col[e] must be in [0, n_in) (n_in = rows of the fixed-k matrix,
 * n_in * ldv < 2^31).  The forward sums each column's terms in edge order
 * with one FFMA rounding per term (k > 32: entries t >= 32 of a group of four
 * edges after the group's first 32 -- a fixed order), the backward in edge
 * order with a product and a sum rounding per term; both deterministic.
 * Columns outside [0, m) are skipped. */
RTK_API int rtk_maxk_spmm_f32(const int64_t *row_ptr, const int32_t *col, const float *aval, int64_t n,
                      const float *vals, const int32_t *idx, const uint8_t *idx8, int64_t ldv, int32_t k,
                      int64_t m, int64_t n_in, float *out, int64_t ldo, void *stream);
RTK_API int rtk_maxk_spmm_backward_f32(const int64_t *row_ptr_t, const int32_t *col_t, const float *aval_t,
                               int64_t n, const float *grad_out, int64_t ldg, const int32_t *idx,
                               const uint8_t *idx8, int64_t ldv, int32_t k, int64_t m, float *grad_vals,
                               void *stream);

/* File-level job: RTKM matrix file -> row top-k on the current CUDA device
 * -> RTKR result file, streamed in chunks of `chunk_rows` rows (0 = ~64 MB):
 * pread into pinned host buffers, H2D, kernel, D2H and pwrite of consecutive
 * chunks overlap (three CUDA streams, double-buffered).  Replaces the
 * reference's load_matrix -> batch_topk -> save_result chain
 * (io.py:46-78, batch.py:105-142; formats SPEC.md:239): magic "RTKM"/"RTKR",
 * u32 version 1, u64 n_rows, u64 n_cols (= k for results), little-endian
 * binary32 payload; the result holds all values then all indices (u32).
 * mode: 0 exact (eps_rel, hard_cap), 1 early stop (max_iter).
 * Unlike the operator entry points this call allocates (device + pinned
 * buffers) and synchronises.  Error precedence follows the reference:
 * RTK_EIO / RTK_EFORMAT / RTK_ETRUNC for the input file, then RTK_ENAN
 * (dims[2] = first row holding a NaN; the partial output is removed), then
 * RTK_EINVAL for k outside [1, n_cols].  dims (nullable) receives
 * {n_rows, n_cols, first_nan_row or -1}. */
RTK_API int rtk_topk_file_f32(const char *matrix_path, const char *result_path, int32_t k, int32_t mode,
                      double eps_rel, int32_t hard_cap, int32_t max_iter, int64_t chunk_rows,
                      int64_t *dims);

/* Thread-local description of the last non-OK return. */
RTK_API const char *rtk_last_error(void);

/* Library ABI version (major*10000 + minor*100 + patch). */
RTK_API int rtk_version(void);

/* The launch configuration the dispatcher picks for an aligned, contiguous
 * 2^20 x m matrix (no traces for modes 0/1; mode 0 = exact, 1 = early stop,
 * 2 = trace) on the current device, without launching: warps per CTA,
 * resident CTAs per SM (occupancy of that kernel instantiation; 1 when no
 * device is present) and rows a warp works on at a time (2 = paired-row
 * kernel, 1 = one row per warp, 0 = the CTA's warps share one row).  For
 * k == m: the elementwise copy (8 warps, 0, 0).  Returns RTK_OK or
 * RTK_EINVAL. */
RTK_API int rtk_launch_shape(int64_t m, int32_t k, int32_t mode, int32_t *warps_per_cta,
                     int32_t *ctas_per_sm, int32_t *rows_per_warp);

#ifdef __cplusplus
}
#endif

#endif /* RTK_H_ */
