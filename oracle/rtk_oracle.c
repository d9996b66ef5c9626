/*
 * rtk_oracle.c -- CPU restatement of the reference row-wise top-k path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path; it may be linked/called only from tests/, from
 * __graft_entry__.smoke() and from bench.py's cpu_baseline / --impl
 * reference arm.  The product library (paper_2409_00822_b200/librtk.so)
 * never links or calls it.
 *
 * Every function restates one function of
 *   /root/reference/pkg/src/rowtopk/_kernels.py
 * literally, including the float64 midpoint rounded once to float32
 * (_kernels.py:72,97) and the float64 loop test (_kernels.py:60,65).
 * Build with -ffp-contract=off and without -ffast-math so every operation is
 * one IEEE-754 round-to-nearest operation, like numba's non-fastmath code.
 *
 * Parity of this oracle with the reference itself is pinned by
 * tests/golden/ (fixtures and digests produced by importing the reference
 * package in the build container, see tests/golden/make_golden.py) and by
 * tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* _kernels.py:19-23 */
enum {
    EXIT_COUNT_EQUALS_K = 1,
    EXIT_INTERVAL_BELOW_EPSILON = 2,
    EXIT_MAX_ITER_REACHED = 3,
    EXIT_HARD_CAP_REACHED = 4,
    EXIT_DEGENERATE_ROW = 5,
};

/* _kernels.py:26-36 -- first-wins strict comparisons. */
static void row_min_max(const float *v, int64_t m, float *mn_out, float *mx_out)
{
    float mn = v[0], mx = v[0];
    for (int64_t i = 1; i < m; ++i) {
        float x = v[i];
        if (x < mn)
            mn = x;
        else if (x > mx)
            mx = x;
    }
    *mn_out = mn;
    *mx_out = mx;
}

/* _kernels.py:39-45 -- inclusive count. */
static int64_t count_ge(const float *v, int64_t m, float t)
{
    int64_t c = 0;
    for (int64_t i = 0; i < m; ++i)
        if (v[i] >= t)
            ++c;
    return c;
}

/* _kernels.py:72 / :97 -- F32((F64(mn) + F64(mx)) * 0.5). */
static float mid_f64(float mn, float mx)
{
    double s = (double)mn + (double)mx;
    return (float)(s * 0.5);
}

/* The float32-only midpoint the CUDA kernels use;
 * exported only so tests can prove it equals mid_f64 on CPU. */
float rtko_mid_f32(float a, float b)
{
    float s = a + b;
    if (isinf(s) && isfinite(a) && isfinite(b)) {
        float ha = a * 0.5f;
        float hb = b * 0.5f;
        return ha + hb;
    }
    return s * 0.5f;
}

float rtko_mid_f64(float a, float b) { return mid_f64(a, b); }

typedef struct {
    float thres, mn, mx;
    int64_t cnt;
    int32_t it;
    int8_t reason;
} search_out;

/* _kernels.py:48-84 (Algorithm 1 with the SPEC exits). */
static search_out exact_search(const float *v, int64_t m, int64_t k, double eps_rel, int32_t hard_cap)
{
    search_out o;
    float mn, mx;
    row_min_max(v, m, &mn, &mx);
    double eps = eps_rel * (double)mx; /* :60 */
    float thres = mn;                  /* :61 */
    int64_t cnt = m;                   /* :62 */
    int32_t it = 0;                    /* :63 */
    for (;;) {
        if (!((double)mx - (double)mn > eps)) { /* :65 */
            o.reason = (it == 0) ? EXIT_DEGENERATE_ROW : EXIT_INTERVAL_BELOW_EPSILON;
            break;
        }
        if (it >= hard_cap) { /* :69 */
            o.reason = EXIT_HARD_CAP_REACHED;
            break;
        }
        it += 1;
        float mid = mid_f64(mn, mx); /* :72 */
        thres = mid;
        cnt = count_ge(v, m, thres);
        if (cnt == k) {
            o.reason = EXIT_COUNT_EQUALS_K;
            break;
        } else if (cnt < k) {
            if (mid == mx) {
                o.reason = EXIT_INTERVAL_BELOW_EPSILON;
                break;
            }
            mx = mid;
        } else {
            if (mid == mn) {
                o.reason = EXIT_INTERVAL_BELOW_EPSILON;
                break;
            }
            mn = mid;
        }
    }
    o.thres = thres;
    o.mn = mn;
    o.mx = mx;
    o.cnt = cnt;
    o.it = it;
    return o;
}

/* _kernels.py:87-103 (Algorithm 2). Returns reason; writes mn/mx/it. */
static int8_t early_search(const float *v, int64_t m, int64_t k, int32_t max_iter,
                           float *mn_out, float *mx_out, int32_t *it_out)
{
    float mn, mx;
    row_min_max(v, m, &mn, &mx);
    if (!(mx > mn)) { /* :94 */
        *mn_out = mn;
        *mx_out = mx;
        *it_out = 0;
        return EXIT_DEGENERATE_ROW;
    }
    for (int32_t i = 0; i < max_iter; ++i) {
        float mid = mid_f64(mn, mx);
        int64_t cnt = count_ge(v, m, mid);
        if (cnt < k)
            mx = mid;
        else
            mn = mid;
    }
    *mn_out = mn;
    *mx_out = mx;
    *it_out = max_iter;
    return EXIT_MAX_ITER_REACHED;
}

/* _kernels.py:106-146 -- first k with v >= thres, else fill from [lo, thres). */
static int64_t select_threshold(const float *v, int64_t m, int64_t k, float thres, float lo,
                                float *out_vals, int32_t *out_idx)
{
    int64_t cnt = count_ge(v, m, thres);
    int64_t j = 0;
    if (cnt >= k) {
        for (int64_t i = 0; i < m; ++i) {
            if (v[i] >= thres) {
                out_idx[j] = (int32_t)i;
                out_vals[j] = v[i];
                if (++j == k)
                    break;
            }
        }
    } else {
        int64_t need = k - cnt, bound = -1, seen = 0;
        for (int64_t i = 0; i < m; ++i) {
            if (lo <= v[i] && v[i] < thres) {
                if (++seen == need) {
                    bound = i;
                    break;
                }
            }
        }
        for (int64_t i = 0; i < m; ++i) {
            float x = v[i];
            if (x >= thres || (i <= bound && lo <= x && x < thres)) {
                out_idx[j] = (int32_t)i;
                out_vals[j] = x;
                if (++j == k)
                    break;
            }
        }
    }
    return j;
}

/* _kernels.py:149-162 */
static void select_exact(const float *v, int64_t m, int64_t k, const search_out *s, int full_precision,
                         float *out_vals, int32_t *out_idx)
{
    float t = s->thres;
    if (s->cnt > k && full_precision && s->reason != EXIT_DEGENERATE_ROW)
        t = s->mx;
    select_threshold(v, m, k, t, s->mn, out_vals, out_idx);
}

static int resolve_threads(int threads)
{
    if (threads <= 0)
        threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    return threads < 1 ? 1 : threads;
}

/* Contiguous near-equal row ranges, one per thread (batch.py:87-102). */
typedef void (*rows_fn)(void *ctx, int64_t a, int64_t b);
typedef struct {
    rows_fn fn;
    void *ctx;
    int64_t a, b;
} range_job;

static void *run_range(void *p)
{
    range_job *j = (range_job *)p;
    j->fn(j->ctx, j->a, j->b);
    return NULL;
}

static void parallel_rows(rows_fn fn, void *ctx, int64_t n, int threads)
{
    threads = resolve_threads(threads);
    if ((int64_t)threads > n)
        threads = (int)(n > 0 ? n : 1);
    if (threads <= 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t tid[256];
    range_job jobs[256];
    if (threads > 256)
        threads = 256;
    for (int t = 0; t < threads; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].a = n * t / threads;
        jobs[t].b = n * (t + 1) / threads;
        if (pthread_create(&tid[t], NULL, run_range, &jobs[t]) != 0) {
            run_range(&jobs[t]);
            tid[t] = 0;
        }
    }
    for (int t = 0; t < threads; ++t)
        if (tid[t])
            pthread_join(tid[t], NULL);
}

static void full_row(const float *row, int64_t m, float *ov, int32_t *oi, int32_t *it, int8_t *rs)
{
    /* _kernels.py:173-179 (k == M shortcut) */
    for (int64_t j = 0; j < m; ++j) {
        ov[j] = row[j];
        oi[j] = (int32_t)j;
    }
    *it = 0;
    *rs = EXIT_DEGENERATE_ROW;
}

typedef struct {
    const float *x;
    int64_t m, ldx, ldo;
    int32_t k, hard_cap, max_iter;
    double eps_rel;
    float *vals;
    int32_t *idx, *iters;
    int8_t *reasons;
} job_args;

/* _kernels.py:165-186 (exact_topk_chunk) over rows [a, b). */
static void exact_rows(void *ctx, int64_t a, int64_t b)
{
    const job_args *j = (const job_args *)ctx;
    int full_precision = (j->eps_rel == 0.0);
    for (int64_t r = a; r < b; ++r) {
        const float *row = j->x + r * j->ldx;
        float *ov = j->vals + r * j->ldo;
        int32_t *oi = j->idx + r * j->ldo;
        int32_t it;
        int8_t rs;
        if ((int64_t)j->k == j->m) {
            full_row(row, j->m, ov, oi, &it, &rs);
        } else {
            search_out s = exact_search(row, j->m, j->k, j->eps_rel, j->hard_cap);
            select_exact(row, j->m, j->k, &s, full_precision, ov, oi);
            it = s.it;
            rs = s.reason;
        }
        if (j->iters)
            j->iters[r] = it;
        if (j->reasons)
            j->reasons[r] = rs;
    }
}

/* _kernels.py:189-214 (early_topk_chunk) over rows [a, b). */
static void early_rows(void *ctx, int64_t a, int64_t b)
{
    const job_args *j = (const job_args *)ctx;
    for (int64_t r = a; r < b; ++r) {
        const float *row = j->x + r * j->ldx;
        float *ov = j->vals + r * j->ldo;
        int32_t *oi = j->idx + r * j->ldo;
        int32_t it;
        int8_t rs;
        if ((int64_t)j->k == j->m) {
            full_row(row, j->m, ov, oi, &it, &rs);
        } else {
            float mn, mx;
            rs = early_search(row, j->m, j->k, j->max_iter, &mn, &mx, &it);
            int64_t c = 0; /* :205-212 */
            for (int64_t i = 0; i < j->m; ++i) {
                if (row[i] >= mn) {
                    oi[c] = (int32_t)i;
                    ov[c] = row[i];
                    if (++c == j->k)
                        break;
                }
            }
        }
        if (j->iters)
            j->iters[r] = it;
        if (j->reasons)
            j->reasons[r] = rs;
    }
}

/* _kernels.py:217-231 (exact_trace_chunk) over rows [a, b). */
static void trace_rows(void *ctx, int64_t a, int64_t b)
{
    const job_args *j = (const job_args *)ctx;
    for (int64_t r = a; r < b; ++r) {
        if ((int64_t)j->k == j->m) {
            j->iters[r] = 0;
            j->reasons[r] = EXIT_DEGENERATE_ROW;
            continue;
        }
        search_out s = exact_search(j->x + r * j->ldx, j->m, j->k, j->eps_rel, j->hard_cap);
        j->iters[r] = s.it;
        j->reasons[r] = s.reason;
    }
}

/* Rows [0, n) of x (row stride ldx); outputs row stride ldo; threads <= 0 = all cores. */
void rtko_exact_topk(const float *x, int64_t n, int64_t m, int64_t ldx, int32_t k, double eps_rel,
                     int32_t hard_cap, float *vals, int32_t *idx, int64_t ldo, int32_t *iters,
                     int8_t *reasons, int threads)
{
    job_args j = {x, m, ldx, ldo, k, hard_cap, 0, eps_rel, vals, idx, iters, reasons};
    parallel_rows(exact_rows, &j, n, threads);
}

void rtko_early_topk(const float *x, int64_t n, int64_t m, int64_t ldx, int32_t k, int32_t max_iter,
                     float *vals, int32_t *idx, int64_t ldo, int32_t *iters, int8_t *reasons,
                     int threads)
{
    job_args j = {x, m, ldx, ldo, k, 0, max_iter, 0.0, vals, idx, iters, reasons};
    parallel_rows(early_rows, &j, n, threads);
}

void rtko_exact_trace(const float *x, int64_t n, int64_t m, int64_t ldx, int32_t k, double eps_rel,
                      int32_t hard_cap, int32_t *iters, int8_t *reasons, int threads)
{
    job_args j = {x, m, ldx, 0, k, hard_cap, 0, eps_rel, NULL, NULL, iters, reasons};
    parallel_rows(trace_rows, &j, n, threads);
}

/* batch.py:37-39 -- index of the first row containing NaN, or -1. */
int64_t rtko_first_nan_row(const float *x, int64_t n, int64_t m, int64_t ldx)
{
    for (int64_t r = 0; r < n; ++r)
        for (int64_t j = 0; j < m; ++j)
            if (isnan(x[r * ldx + j]))
                return r;
    return -1;
}

/* Single-row pieces (_kernels.py:26-45), for unit tests. */
void rtko_row_min_max(const float *v, int64_t m, float *mn, float *mx) { row_min_max(v, m, mn, mx); }
int64_t rtko_count_ge(const float *v, int64_t m, float t) { return count_ge(v, m, t); }

int rtko_max_threads(void) { return resolve_threads(0); }

/* Bulk proof helper: number of pairs (a[i], b[i]) (bit patterns) where the
 * float32-only midpoint differs bitwise from the reference f64 midpoint.
 * NaN inputs are skipped (NaN never reaches a midpoint for valid input). */
int64_t rtko_mid_mismatches(const uint32_t *a, const uint32_t *b, int64_t n)
{
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        float x, y;
        memcpy(&x, &a[i], 4);
        memcpy(&y, &b[i], 4);
        if (isnan(x) || isnan(y))
            continue;
        float p = rtko_mid_f32(x, y), q = mid_f64(x, y);
        uint32_t pb, qb;
        memcpy(&pb, &p, 4);
        memcpy(&qb, &q, 4);
        if (pb != qb && !(isnan(p) && isnan(q)))
            ++bad;
    }
    return bad;
}
