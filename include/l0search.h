/*
 * l0search.h -- C ABI of the B200-native SO / l0 descriptor search.
 *
 * The reference (descsearch 0.1.0, /root/reference/pkg) is a Python package
 * whose only native code is four numba kernels; it has no FFI.  Its operator
 * boundary for this path is the Python function
 *
 *     descsearch.search.l0_search(subspace, property_values, task_slices,
 *                                 config, workers, task_labels, stats)
 *                                                      search.py:202-322
 *
 * and its companions fit_tuple (search.py:136-171) and the kernels
 * score_tuples / fit_tuple_kernel / fill_combinations (lsq.py:113-215).
 * The Python host package paper_2502_20072_b200 mirrors that API and binds
 * the entry points below with ctypes.
 *
 * Conventions:
 *   - every function returns an int status (L0S_OK == 0); l0s_last_error()
 *     gives a per-thread message for the last failure;
 *   - the caller owns every in/out buffer; the context owns device memory,
 *     streams and events;
 *   - a context is bound to one CUDA device and is not thread-safe; calls
 *     block until their results are in the caller's buffers.
 *   - no CPU fallback: without a usable sm_100 device l0s_create fails with
 *     L0S_ENODEV.
 */
#ifndef L0SEARCH_H
#define L0SEARCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define L0S_OK 0
#define L0S_EINVAL 1    /* maps to ValueError                          */
#define L0S_ECAPACITY 2 /* maps to descsearch.errors.CapacityError      */
#define L0S_ECUDA 3     /* maps to RuntimeError                         */
#define L0S_ENOMEM 4    /* device allocation failed -> RuntimeError     */
#define L0S_ENODEV 5    /* no usable B200 / sm_100 device              */
#define L0S_ESTATE 6    /* call order violated (e.g. search before stage) */

#define L0S_PREC_FP64 0
#define L0S_PREC_FP32 1

/* search modes (l0s_search 'mode') */
#define L0S_MODE_AUTO 0  /* screened Gram path when it applies, exact otherwise   */
#define L0S_MODE_FAST 1  /* force the screened Gram path (n in {2,3,4}, T <= 8)   */
#define L0S_MODE_EXACT 2 /* score every tuple with the bit-exact Householder kernel */

typedef struct l0s_ctx l0s_ctx;

/* Throughput / diagnostics bookkeeping (superset of search.SearchStats, search.py:45-56). */
typedef struct {
    int64_t n_tuples;        /* tuples in [rank_begin, rank_end)                      */
    double ms_total;         /* device time of the whole search (events)              */
    double ms_fit;           /* screened fit kernel(s)                                */
    double ms_exact;         /* bit-exact kernels (refit / ill / exact mode)          */
    double ms_gram;          /* stage + Gram, set by l0s_stage                        */
    double theta;            /* final global screening threshold                      */
    int64_t n_candidates;    /* screened candidates refit exactly                     */
    int64_t n_ill;           /* tuples routed to the exact kernel by conditioning     */
    int64_t n_rescan;        /* certification rescans                                 */
    int64_t n_fit_launches;  /* kernel launches of the screened fit                   */
    int64_t n_launches;      /* all kernel launches of this search                    */
    int32_t mode_used;       /* L0S_MODE_FAST or L0S_MODE_EXACT                       */
    int32_t certified;       /* 1 when the top-k set is proven exact                  */
    double margin;           /* lb(K')-th minus k-th exact score at certification     */
    double ms_qr;            /* QR screen of the uncertifiable tuples                 */
    int64_t n_ill_refit;     /* of those, refit bit-exactly                           */
    double ms_gram_kernel;   /* the Gram kernel alone (device-resident, unchunked stage) */
    double ms_records;       /* final records: refit of kept tuples not already refit (excluded from
                                SearchStats.seconds like the reference's per-model fit_tuple)    */
    int64_t n_eval;          /* task-tuple evaluations the screened sweep executed (one (i, j, k, task)
                                bound term; the physical work behind the roofline)             */
    int64_t n_screen;        /* tile-screen tests of the n = 3 sweep (one warp: 32 j x P pairs bounded
                                over a group of i-tiles or one tile; fit3.cu tile_screen)      */
} l0s_stats;

const char *l0s_last_error(void);
int l0s_version(void);

/* Device discovery: number of CUDA devices (0 when none). */
int l0s_device_count(int *count);

/* Context on one device (replaces the per-call thread pool of search.py:258-301). */
int l0s_create(int device, l0s_ctx **out);
int l0s_destroy(l0s_ctx *ctx);

/*
 * Stage one problem on the device (replaces search._prepare, search.py:113-127,
 * and adds the Gram precompute).
 *   values : (m, s) float64, row-major, samples in the caller's original order
 *   y      : (s,)   float64
 *   perm   : (s,)   int64, concatenation of the task slices in task order
 *   bounds : (ntasks+1,) int64 task boundaries on the permuted axis
 *   precision : L0S_PREC_FP64 / L0S_PREC_FP32 (values and y are rounded to
 *            float32 first, as _prepare does, search.py:125-126)
 *   is_device : 1 when values / y / perm are device pointers on this context's device
 * The Gram (normalized, per-task centered, fp64 DMMA) is built here.
 */
int l0s_stage(l0s_ctx *ctx, const double *values, int64_t m, int64_t s, const double *y,
              const int64_t *perm, const int64_t *bounds, int ntasks, int precision,
              int is_device);

/*
 * Multi-GPU staging (one process per GPU): every rank stages the whole problem but computes
 * only its shard of the Gram -- a contiguous range of the T x (upper-triangle 64 x 64 block)
 * order -- into `pack` (device buffer of l0s_gram_shard_size doubles).  The caller all-gathers
 * the packs in rank order (NCCL over NVLink) and hands the gathered buffer (nshards x pack
 * doubles, device memory) to l0s_stage_finish, which scatters it into the full Gram and
 * completes the stage.  nshards == 1 is l0s_stage.  (search.py:113-127 + the Gram precompute,
 * split across GPUs; no reference counterpart -- the reference is single-process.)
 */
int l0s_gram_shard_size(int64_t m, int ntasks, int nshards, int64_t *out_doubles);

/*
 * Append m_new feature rows (host, (m_new, s) float64, the caller's sample
 * order) to the problem of the previous l0s_stage (host inputs), as the
 * pipeline's subspace grows between dimensions (screening.py:197-198,
 * pipeline.py:181-240): only the new rows are copied; the result is the stage
 * of the concatenated matrix.  L0S_ESTATE unless the context holds a
 * completed stage from host inputs.
 */
int l0s_stage_append(l0s_ctx *ctx, const double *rows, int64_t m_new);

/*
 * One of nparts disjoint parts of the whole search (multi-GPU: part = rank).
 * The screened path takes every nparts-th unit of its (longest-first) unit
 * table, so ill-conditioned tuples that cluster in one rank range (C4) spread
 * over all parts; otherwise part p is the contiguous rank range
 * [p N / nparts, (p+1) N / nparts) (search.py:266-271).  Every part returns
 * its own exact top list; the (score, rank) merge of all parts is the whole
 * search's (search.py:303).  The path is chosen on the whole problem, so all
 * parts agree.
 */
int l0s_search_part(l0s_ctx *ctx, int n, int64_t keep, int part, int nparts, int mode,
                    double *out_scores, int64_t *out_ranks, double *out_coef, double *out_ssr,
                    int64_t *out_count, l0s_stats *stats);

/*
 * Cross-part exchange for l0s_search_part (multi-GPU; no reference counterpart: the reference's
 * workers share one process and merge at the end, search.py:258-304).  When set, every
 * screened search part calls fn exactly once, after refitting its first candidates and before
 * certifying: scores = the part's best exact scores so far (ascending, count <= keep).  fn must
 * return an upper bound on the whole search's keep-th score -- a collective: the keep-th of the
 * union of every part's list (all-gather + merge), or +inf.  The part then certifies against
 * it instead of its own keep-th, so a part holding dense near-ties need not rescan for tuples
 * other parts have already beaten.  A part that fails before the exchange leaves the others
 * waiting in fn: the caller's collective must handle that (the group API's does).  fn == NULL
 * clears it.
 */
typedef double (*l0s_exchange_fn)(const double *scores, int64_t count, void *user);
int l0s_set_part_exchange(l0s_ctx *ctx, l0s_exchange_fn fn, void *user);

/*
 * l0s_stage / l0s_stage_append with the feature rows given as m (m_new) host
 * pointers to s float64 each -- a SelectedSubspace's entry arrays
 * (screening.py:165-198) copied row by row, never stacked on the host
 * (values_matrix, screening.py:191-195, costs a host copy of the whole
 * matrix per call).
 */
int l0s_stage_rows(l0s_ctx *ctx, const double *const *rows, int64_t m, int64_t s, const double *y,
                   const int64_t *perm, const int64_t *bounds, int ntasks, int precision);
int l0s_stage_append_rows(l0s_ctx *ctx, const double *const *rows, int64_t m_new);

/*
 * Final-rung candidates on the device (generation.iter_final_rung,
 * generation.py:331-393; values: expressions.apply_operator_values,
 * expressions.py:168-192; validity: generation._validity_mask, :107-118).
 *
 * l0s_gen_pool: the pool's value rows (host, (n_pool, s), float64 or, with
 *   fp32 = 1, float32 -- the pool's dtype), resident until the next call.
 * l0s_gen_eval: candidates c < count of one operator kind (L0S_GEN_*):
 *   children pi[c], pj[c] (pj NULL or -1 for unary kinds); kind
 *   L0S_GEN_VALUES takes the rows from `values` ((count, s), pool dtype)
 *   instead.  Writes out_valid[c] (the reference's validity rule with limits
 *   min_abs / max_abs / dedup_tol compared in the pool's dtype) and
 *   out_hash[2c..2c+1] (128-bit fingerprint of float64(v) rounded to `tol`,
 *   half to even, -0 == +0: equal iff the rounded vectors are equal, up to
 *   hash collisions).  The values stay on the device (fp64).
 * l0s_gen_take: rows[] of the last evaluation into a compact fp64 device
 *   block (*dev_out, valid until the next l0s_gen_* call; feed it to
 *   l0s_sis_scores with is_device = 1) and, if host_out, to the host in the
 *   pool's dtype.
 * l0s_gen_fetch: rows[] of the taken block to the host (pool dtype).
 */
#define L0S_GEN_COPY 0
#define L0S_GEN_ADD 1
#define L0S_GEN_SUB 2
#define L0S_GEN_MUL 3
#define L0S_GEN_DIV 4
#define L0S_GEN_ABS_DIFF 5
#define L0S_GEN_SQRT 6
#define L0S_GEN_SQ 7
#define L0S_GEN_CB 8
#define L0S_GEN_INV 9
#define L0S_GEN_ABS 10
#define L0S_GEN_VALUES 11
int l0s_gen_pool(l0s_ctx *ctx, const void *values, int64_t n_pool, int64_t s, int fp32);
int l0s_gen_eval(l0s_ctx *ctx, int kind, const int32_t *pi, const int32_t *pj, int64_t count,
                 const void *values, double tol, double min_abs, double max_abs, double dedup_tol,
                 uint8_t *out_valid, uint64_t *out_hash);
int l0s_gen_take(l0s_ctx *ctx, const int32_t *rows, int64_t count, void *host_out,
                 const double **dev_out);
int l0s_gen_fetch(l0s_ctx *ctx, const int32_t *rows, int64_t count, void *host_out);
int l0s_stage_shard(l0s_ctx *ctx, const double *values, int64_t m, int64_t s, const double *y,
                    const int64_t *perm, const int64_t *bounds, int ntasks, int precision,
                    int is_device, int shard, int nshards, double *pack);
int l0s_stage_finish(l0s_ctx *ctx, const double *gathered);

/*
 * Exhaustive search over tuple ranks [rank_begin, rank_end) of C(m, n)
 * (search.l0_search's scan + merge, search.py:233-304).  Writes the best
 * min(keep, #finite) tuples ordered by (score, rank); scores and ssr are
 * bit-identical to the reference's score_tuples / fit_tuple_kernel.
 *   out_scores : (keep,) float64   score = sum_task ssr / s (lsq.py:153-156)
 *   out_ranks  : (keep,) int64
 *   out_coef   : (keep, ntasks, n+1) float64 (working-dtype values widened)
 *   out_ssr    : (keep, ntasks) float64
 *   out_count  : number written
 */
int l0s_search(l0s_ctx *ctx, int n, int64_t keep, int64_t rank_begin, int64_t rank_end,
               int mode, double *out_scores, int64_t *out_ranks, double *out_coef,
               double *out_ssr, int64_t *out_count, l0s_stats *stats);

/*
 * Bit-exact fits of explicit tuples (fit_tuple_kernel, lsq.py:159-192, for
 * many tuples at once).  tuples: (count, n) int64 strictly increasing.
 *   out_ok    : (count,) int32
 *   out_score : (count,) float64  score_tuples value (+inf when deficient)
 *   out_coef  : (count, ntasks, n+1) float64;  out_ssr : (count, ntasks)
 */
int l0s_fit_tuples(l0s_ctx *ctx, int n, const int64_t *tuples, int64_t count, int32_t *out_ok,
                   double *out_score, double *out_coef, double *out_ssr);

/*
 * Screened lower bounds for explicit tuples (diagnostics / tests): the value
 * the fit kernel compares against its threshold, lb <= exact score, with
 * flag bit0 = conditioning check passed, bit1 = reference rank rule certain.
 */
int l0s_screen_tuples(l0s_ctx *ctx, int n, const int64_t *tuples, int64_t count, double *out_lb,
                      int32_t *out_flags);

/*
 * SIS projection scores (screening._chunk_scores, screening.py:126-155),
 * bit-identical to the reference's fixed-shape pairwise sums.
 *   l0s_sis_prepare: targets (R x s) float64 in dataset sample order (R <= 8), the task
 *                    slices as perm (concatenated, int64) + bounds (ntasks+1)
 *   l0s_sis_scores : F (k x s) float64 feature rows (host, or device with is_device=1)
 *                    -> out (k) float64 host: clip(max_r sum_t w_t |pearson_t|, 0, 1)
 */
int l0s_sis_prepare(l0s_ctx *ctx, const double *targets, int R, int64_t s, const int64_t *perm,
                    const int64_t *bounds, int ntasks);
int l0s_sis_scores(l0s_ctx *ctx, const double *F, int64_t k, int is_device, double *out);

/* Gram method of subsequent stages: AUTO (INT8 Ozaki on tcgen05 for fp64 problems with
 * m >= 256, DMMA otherwise or when the INT8 error bound is too loose), DMMA (fp64 tensor),
 * OZAKI (INT8 whenever possible). */
#define L0S_GRAM_AUTO 0
#define L0S_GRAM_DMMA 1
#define L0S_GRAM_OZAKI 2
int l0s_set_gram_mode(l0s_ctx *ctx, int mode);
/* Per-task entry error bound of the staged Gram (ntasks values) and whether it is the INT8 one. */
int l0s_stage_info(l0s_ctx *ctx, double *eta_out, int *ozaki_out);
/* Rows of the last INT8 Gram whose own error term exceeded the screen's limit (spiky rows, max |z|
 * close to 1; e.g. a Gaussian property): up to 64 of them were recomputed in fp64 and left out of
 * eta; with more, the whole Gram was recomputed on DMMA (l0s_stage_info then reports ozaki 0). */
int l0s_stage_loose_rows(l0s_ctx *ctx, int *out_count);
/* Device times (ms) of the last stage when its inputs were device-resident (unchunked):
 * [gather (search._prepare's permutation + cast), normalize (+ INT8 digits), Gram, feature
 * flags]; zeros after a chunked host stage. */
int l0s_stage_timings(l0s_ctx *ctx, double *out_ms);

/* Diagnostics: the device QR screen (warp TSQR) of explicit tuples: pooled score sum_t ssr_t / s
 * and the smallest rank-rule ratio min_j |R_jj| / max_j |R_jj| over the tasks. */
int l0s_qr_tuples(l0s_ctx *ctx, int n, const int64_t *tuples, int64_t count, double *out_score,
                  double *out_ratio);

/*
 * Residual targets of the next SIS round (models.residuals / predict, models.py:44-83) from the
 * staged inputs: out[c][i] = y[i] - (coef[c][t][n] + sum_k coef[c][t][k] x_{tup[c][k]}[i]) for every
 * sample i (caller's order) of task t, numpy's operation order.  tuples (count, n) index the
 * staged features; coef (count, ntasks, n+1) float64 (a Model's coefficients); out (count, s).
 */
int l0s_residuals(l0s_ctx *ctx, int n, const int64_t *tuples, const double *coef, int64_t count,
                  double *out);

/* Copy of the staged normalized Gram of one task ((m+1) x (m+1), last row/col = y). */
int l0s_get_gram(l0s_ctx *ctx, int task, double *out);

/* Unranking helpers on the device's binomial table (search.py:66-104). */
int l0s_unrank(int64_t rank, int64_t m, int n, int64_t *out_tuple);
int l0s_rank(const int64_t *tuple, int64_t m, int n, int64_t *out_rank);
int l0s_count(int64_t m, int n, int64_t *out_count); /* C(m,n); L0S_ECAPACITY if >= 2^63 */

/* Microbenchmarks used by bench.py for the roofline denominator. */
int l0s_fp64_peak(l0s_ctx *ctx, double *out_tflops);
/* Worst relative error of the screen's fast reciprocal over `count` hashed doubles
 * (the screen assumes <= 2^-17; tests/test_gpu_parity.py::test_rcp_fast_bound checks it). */
int l0s_rcp_check(int64_t count, double *out_max_rel);

/*
 * The streamed last rung's value dedup on the device (the reference's ordered walk,
 * generation.py:364-385, for operator lists without repeated kinds, where the key test
 * cannot fire).  l0s_gen_dedup_reset seeds a device set with the pool's 128-bit fingerprints
 * (count x 2 uint64, as l0s_gen_eval writes them); l0s_gen_dedup marks, for the candidates of
 * the last l0s_gen_eval, out_kept[x] = 1 iff x is valid and no earlier candidate of the stream
 * (or pool entry) has its fingerprint, and adds the kept fingerprints to the set.
 */
int l0s_gen_dedup_reset(l0s_ctx *ctx, const uint64_t *seed, int64_t count);
int l0s_gen_dedup(l0s_ctx *ctx, uint8_t *out_kept, int64_t *out_count);

/*
 * Several devices in one process (the reference's in-process `workers`, search.py:258-304):
 * one context per device (devices may repeat), one host thread per device.
 *   l0s_group_stage  : device g uploads row block g of the inputs (values: (m, s) row-major, or
 *                      rows: m host pointers, exactly one non-null; pageable or pinned), the
 *                      blocks are exchanged device to device (cudaMemcpyPeerAsync), every device
 *                      stages the whole problem (l0s_stage on its copy);
 *   l0s_group_search : device g searches part g (l0s_search_part); the exact per-part top lists
 *                      merge by (score, rank) (search.py:303); outputs as l0s_search, stats
 *                      summed (counts) or maxed (times) over the devices.
 */
typedef struct l0s_group l0s_group;
int l0s_group_create(int ndev, const int *devices, l0s_group **out);
int l0s_group_destroy(l0s_group *group);
int l0s_group_size(l0s_group *group, int *out);
int l0s_group_ctx(l0s_group *group, int member, l0s_ctx **out);
int l0s_group_stage(l0s_group *group, const double *values, const double *const *rows, int64_t m,
                    int64_t s, const double *y, const int64_t *perm, const int64_t *bounds,
                    int ntasks, int precision);
int l0s_group_search(l0s_group *group, int n, int64_t keep, int mode, double *out_scores,
                     int64_t *out_ranks, double *out_coef, double *out_ssr, int64_t *out_count,
                     l0s_stats *stats);

#ifdef __cplusplus
}
#endif

#endif /* L0SEARCH_H */
