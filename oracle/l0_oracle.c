/*
 * l0_oracle.c -- CPU restatement of the reference's l0 (SO) search kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg use it, as the checker and as the timed
 * CPU baseline.  Parity is pinned by tests/test_oracle.py against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py runs
 * descsearch's numba kernels in the build container).
 *
 * Restated functions (reference = /root/reference/pkg/src/descsearch/lsq.py):
 *   orc_solve_f64 / orc_solve_f32  <- _solve_inplace      lsq.py:61-110
 *   orc_score_tuples               <- score_tuples        lsq.py:113-156
 *   orc_fit_tuple                  <- fit_tuple_kernel    lsq.py:159-192
 *   orc_fill_combinations          <- fill_combinations   lsq.py:195-215
 *   orc_scan                       <- search._scan_range + worker pool
 *                                     (search.py:174-199, 258-304), with an
 *                                     exact (score, rank) top-keep per thread.
 *
 * Arithmetic contract (what makes the results bit-identical to numba, which
 * compiles without fast-math and does not contract a*b+c): build with
 * -O2 -ffp-contract=off, no -ffast-math; every reduction is a sequential loop
 * in the reference's order; sqrt and '/' are IEEE.  The float32 path keeps
 * numba's mixed typing: products of two float32 values are rounded to float32,
 * the Householder norms / dots / ssr accumulate in float64 (their
 * accumulators are initialised with the float64 literal 0.0), updated matrix
 * entries are rounded back to float32 on store, and the back-substitution runs
 * entirely in float32.
 *
 * The scratch matrix is column-major here (column c of task rows starts at
 * A + c*ld); the reference's is row-major.  Storage order does not change any
 * rounding.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

/* ---------------- Householder solve (lsq.py:61-110) ---------------- */

static int orc_solve_f64(double *A, int64_t ld, int64_t rows, int p, double tol,
                         double *coef, double *ssr_out)
{
    double maxdiag = 0.0;
    int ok = 1;
    for (int j = 0; j < p; ++j) {
        double *aj = A + (int64_t)j * ld;
        double nrm2 = 0.0;
        for (int64_t i = j; i < rows; ++i)
            nrm2 += aj[i] * aj[i];
        double nrm = sqrt(nrm2);
        if (nrm == 0.0) {
            ok = 0;
            continue;
        }
        double alpha = (aj[j] >= 0) ? -nrm : nrm;
        double vj = aj[j] - alpha;
        double vtv = nrm2 - aj[j] * aj[j] + vj * vj;
        aj[j] = vj;
        for (int c = j + 1; c <= p; ++c) {
            double *ac = A + (int64_t)c * ld;
            double w = 0.0;
            for (int64_t i = j; i < rows; ++i)
                w += aj[i] * ac[i];
            double fac = 2.0 * w / vtv;
            for (int64_t i = j; i < rows; ++i)
                ac[i] -= fac * aj[i];
        }
        aj[j] = alpha;
        double a = fabs(alpha);
        if (a > maxdiag)
            maxdiag = a;
    }
    if (ok) {
        for (int j = 0; j < p; ++j)
            if (fabs(A[(int64_t)j * ld + j]) < tol * maxdiag)
                ok = 0;
    }
    if (!ok) {
        *ssr_out = 0.0;
        return 0;
    }
    const double *rhs = A + (int64_t)p * ld;
    for (int j = p - 1; j >= 0; --j) {
        double acc = rhs[j];
        for (int c = j + 1; c < p; ++c)
            acc -= A[(int64_t)c * ld + j] * coef[c];
        coef[j] = acc / A[(int64_t)j * ld + j];
    }
    double ssr = 0.0;
    for (int64_t i = p; i < rows; ++i)
        ssr += rhs[i] * rhs[i];
    *ssr_out = ssr;
    return 1;
}

static int orc_solve_f32(float *A, int64_t ld, int64_t rows, int p, double tol,
                         float *coef, double *ssr_out)
{
    double maxdiag = 0.0;
    int ok = 1;
    for (int j = 0; j < p; ++j) {
        float *aj = A + (int64_t)j * ld;
        double nrm2 = 0.0;
        for (int64_t i = j; i < rows; ++i) {
            float pr = aj[i] * aj[i];
            nrm2 += (double)pr;
        }
        double nrm = sqrt(nrm2);
        if (nrm == 0.0) {
            ok = 0;
            continue;
        }
        double alpha = (aj[j] >= 0) ? -nrm : nrm;
        double vj = (double)aj[j] - alpha;
        float djj = aj[j] * aj[j];
        double vtv = nrm2 - (double)djj + vj * vj;
        aj[j] = (float)vj;
        for (int c = j + 1; c <= p; ++c) {
            float *ac = A + (int64_t)c * ld;
            double w = 0.0;
            for (int64_t i = j; i < rows; ++i) {
                float pr = aj[i] * ac[i];
                w += (double)pr;
            }
            double fac = 2.0 * w / vtv;
            for (int64_t i = j; i < rows; ++i)
                ac[i] = (float)((double)ac[i] - fac * (double)aj[i]);
        }
        aj[j] = (float)alpha;
        double a = fabs(alpha);
        if (a > maxdiag)
            maxdiag = a;
    }
    if (ok) {
        for (int j = 0; j < p; ++j)
            if ((double)fabsf(A[(int64_t)j * ld + j]) < tol * maxdiag)
                ok = 0;
    }
    if (!ok) {
        *ssr_out = 0.0;
        return 0;
    }
    const float *rhs = A + (int64_t)p * ld;
    for (int j = p - 1; j >= 0; --j) {
        float acc = rhs[j];
        for (int c = j + 1; c < p; ++c) {
            float pr = A[(int64_t)c * ld + j] * coef[c];
            acc = acc - pr;
        }
        coef[j] = acc / A[(int64_t)j * ld + j];
    }
    double ssr = 0.0;
    for (int64_t i = p; i < rows; ++i) {
        float pr = rhs[i] * rhs[i];
        ssr += (double)pr;
    }
    *ssr_out = ssr;
    return 1;
}

/* ---------------- one tuple, all tasks ---------------- */

typedef struct {
    const void *values; /* (m, s) row-major, task-contiguous columns */
    int is_f32;
    int64_t s;
    const void *y; /* (s,) same dtype as values */
    const int64_t *bounds; /* (ntasks+1,) */
    int ntasks;
    double tol;
} orc_problem;

static int64_t max_rows(const orc_problem *P)
{
    int64_t mr = 0;
    for (int t = 0; t < P->ntasks; ++t) {
        int64_t r = P->bounds[t + 1] - P->bounds[t];
        if (r > mr)
            mr = r;
    }
    return mr;
}

/* Fill the scratch for one task and solve.  coef (p) is in the working dtype. */
static int solve_task(const orc_problem *P, void *scratch, int64_t ld, const int64_t *tup, int n,
                      int task, void *coef, double *ssr)
{
    int64_t lo = P->bounds[task];
    int64_t rows = P->bounds[task + 1] - lo;
    int p = n + 1;
    if (P->is_f32) {
        float *A = (float *)scratch;
        const float *v = (const float *)P->values;
        const float *y = (const float *)P->y;
        for (int k = 0; k < n; ++k) {
            const float *row = v + tup[k] * P->s + lo;
            memcpy(A + (int64_t)k * ld, row, (size_t)rows * sizeof(float));
        }
        for (int64_t i = 0; i < rows; ++i) {
            A[(int64_t)n * ld + i] = 1.0f;
            A[(int64_t)p * ld + i] = y[lo + i];
        }
        return orc_solve_f32(A, ld, rows, p, P->tol, (float *)coef, ssr);
    } else {
        double *A = (double *)scratch;
        const double *v = (const double *)P->values;
        const double *y = (const double *)P->y;
        for (int k = 0; k < n; ++k) {
            const double *row = v + tup[k] * P->s + lo;
            memcpy(A + (int64_t)k * ld, row, (size_t)rows * sizeof(double));
        }
        for (int64_t i = 0; i < rows; ++i) {
            A[(int64_t)n * ld + i] = 1.0;
            A[(int64_t)p * ld + i] = y[lo + i];
        }
        return orc_solve_f64(A, ld, rows, p, P->tol, (double *)coef, ssr);
    }
}

/* score_tuples (lsq.py:113-156): out[t] = sum_task ssr / s, +inf if any task is deficient. */
static double score_one(const orc_problem *P, void *scratch, int64_t ld, const int64_t *tup, int n,
                        void *coef)
{
    double total = 0.0;
    for (int task = 0; task < P->ntasks; ++task) {
        double ssr;
        if (!solve_task(P, scratch, ld, tup, n, task, coef, &ssr))
            return INFINITY;
        total += ssr;
    }
    return total / (double)P->s;
}

static size_t elem_size(const orc_problem *P) { return P->is_f32 ? sizeof(float) : sizeof(double); }

ORC_EXPORT void orc_score_tuples(const void *values, int is_f32, int64_t s, const void *y,
                                 const int64_t *bounds, int ntasks, const int64_t *tuples,
                                 int64_t count, int n, double tol, double *out)
{
    orc_problem P = {values, is_f32, s, y, bounds, ntasks, tol};
    int64_t ld = max_rows(&P);
    if (ld < 1)
        ld = 1;
    void *scratch = malloc((size_t)ld * (size_t)(n + 2) * elem_size(&P));
    void *coef = malloc((size_t)(n + 1) * elem_size(&P));
    for (int64_t t = 0; t < count; ++t)
        out[t] = score_one(&P, scratch, ld, tuples + t * n, n, coef);
    free(scratch);
    free(coef);
}

/* fit_tuple_kernel (lsq.py:159-192). coef_out (ntasks, n+1) in the working dtype. */
ORC_EXPORT int orc_fit_tuple(const void *values, int is_f32, int64_t s, const void *y,
                             const int64_t *bounds, int ntasks, const int64_t *tup, int n,
                             double tol, void *coef_out, double *ssr_out)
{
    orc_problem P = {values, is_f32, s, y, bounds, ntasks, tol};
    int64_t ld = max_rows(&P);
    if (ld < 1)
        ld = 1;
    int p = n + 1;
    void *scratch = malloc((size_t)ld * (size_t)(n + 2) * elem_size(&P));
    int ok = 1;
    for (int task = 0; task < ntasks && ok; ++task) {
        void *row = (char *)coef_out + (size_t)task * (size_t)p * elem_size(&P);
        double ssr;
        if (!solve_task(&P, scratch, ld, tup, n, task, row, &ssr))
            ok = 0;
        else
            ssr_out[task] = ssr;
    }
    free(scratch);
    return ok;
}

/* fill_combinations (lsq.py:195-215): lexicographic successor walk, cursor advanced in place. */
ORC_EXPORT void orc_fill_combinations(int64_t *cur, int n, int64_t m, int64_t *out, int64_t count)
{
    for (int64_t t = 0; t < count; ++t) {
        memcpy(out + t * n, cur, (size_t)n * sizeof(int64_t));
        int j = n - 1;
        while (j >= 0 && cur[j] == m - n + j)
            --j;
        if (j < 0)
            break;
        cur[j] += 1;
        for (int k = j + 1; k < n; ++k)
            cur[k] = cur[k - 1] + 1;
    }
}

/* ---------------- ranks (search.py:59-104) ---------------- */

/* C(a, b) saturated at INT64_MAX. */
ORC_EXPORT int64_t orc_binom(int64_t a, int64_t b)
{
    if (b < 0 || a < 0 || b > a)
        return 0;
    if (b > a - b)
        b = a - b;
    unsigned __int128 r = 1;
    for (int64_t i = 1; i <= b; ++i) {
        r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
        if (r > (unsigned __int128)INT64_MAX)
            return INT64_MAX;
    }
    return (int64_t)r;
}

ORC_EXPORT void orc_unrank(int64_t rank, int64_t m, int n, int64_t *out)
{
    int64_t r = rank, e = 0;
    for (int k = 0; k < n; ++k) {
        int remaining = n - k - 1;
        for (;;) {
            int64_t c = orc_binom(m - 1 - e, remaining);
            if (r < c)
                break;
            r -= c;
            ++e;
        }
        out[k] = e;
        ++e;
    }
}

/* ---------------- threaded exhaustive scan (search.py:174-304) ---------------- */

typedef struct {
    const orc_problem *P;
    int64_t m;
    int n;
    int64_t begin, end;
    int keep;
    double *best_s;
    int64_t *best_r;
    int nbest;
} scan_job;

/* insert (sc, rk) into the ascending (score, rank) list of capacity keep */
static void topk_insert(double *bs, int64_t *br, int *nb, int keep, double sc, int64_t rk)
{
    int cnt = *nb;
    if (cnt == keep) {
        if (sc > bs[cnt - 1] || (sc == bs[cnt - 1] && rk > br[cnt - 1]))
            return;
        --cnt;
    }
    int pos = cnt;
    while (pos > 0 && (bs[pos - 1] > sc || (bs[pos - 1] == sc && br[pos - 1] > rk))) {
        bs[pos] = bs[pos - 1];
        br[pos] = br[pos - 1];
        --pos;
    }
    bs[pos] = sc;
    br[pos] = rk;
    *nb = cnt + 1;
}

static void *scan_worker(void *arg)
{
    scan_job *J = (scan_job *)arg;
    const orc_problem *P = J->P;
    int n = J->n;
    int64_t ld = max_rows(P);
    if (ld < 1)
        ld = 1;
    void *scratch = malloc((size_t)ld * (size_t)(n + 2) * elem_size(P));
    void *coef = malloc((size_t)(n + 1) * elem_size(P));
    int64_t cur[64], tup[64];
    J->nbest = 0;
    if (J->begin < J->end) {
        orc_unrank(J->begin, J->m, n, cur);
        for (int64_t rk = J->begin; rk < J->end; ++rk) {
            orc_fill_combinations(cur, n, J->m, tup, 1);
            double sc = score_one(P, scratch, ld, tup, n, coef);
            if (isfinite(sc))
                topk_insert(J->best_s, J->best_r, &J->nbest, J->keep, sc, rk);
        }
    }
    free(scratch);
    free(coef);
    return NULL;
}

/* Scores ranks [rank_begin, rank_end) on nthreads host threads (disjoint contiguous
 * sub-ranges), returns the best `keep` finite (score, rank) pairs sorted ascending.
 * Returns the number written. */
ORC_EXPORT int orc_scan(const void *values, int is_f32, int64_t s, const void *y,
                        const int64_t *bounds, int ntasks, int64_t m, int n, double tol,
                        int64_t rank_begin, int64_t rank_end, int keep, int nthreads,
                        double *out_scores, int64_t *out_ranks)
{
    if (n < 1 || n > 64 || keep < 1)
        return -1;
    if (nthreads < 1)
        nthreads = 1;
    orc_problem P = {values, is_f32, s, y, bounds, ntasks, tol};
    scan_job *jobs = calloc((size_t)nthreads, sizeof(scan_job));
    pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t total = rank_end - rank_begin;
    for (int w = 0; w < nthreads; ++w) {
        jobs[w].P = &P;
        jobs[w].m = m;
        jobs[w].n = n;
        jobs[w].begin = rank_begin + (total * w) / nthreads;
        jobs[w].end = rank_begin + (total * (w + 1)) / nthreads;
        jobs[w].keep = keep;
        jobs[w].best_s = malloc((size_t)keep * sizeof(double));
        jobs[w].best_r = malloc((size_t)keep * sizeof(int64_t));
        pthread_create(&th[w], NULL, scan_worker, &jobs[w]);
    }
    int nb = 0;
    for (int w = 0; w < nthreads; ++w) {
        pthread_join(th[w], NULL);
        for (int i = 0; i < jobs[w].nbest; ++i)
            topk_insert(out_scores, out_ranks, &nb, keep, jobs[w].best_s[i], jobs[w].best_r[i]);
        free(jobs[w].best_s);
        free(jobs[w].best_r);
    }
    free(jobs);
    free(th);
    return nb;
}
