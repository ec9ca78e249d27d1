// kernels.h -- host-side launchers shared between the translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <vector>

namespace l0s {

// ---- staging (stage.cu) ----
// Gather + cast (search._prepare, search.py:113-127): Xp[f][i] = W(values[f][perm[i]]),
// yp[i] = W(y[perm[i]]), W = double (fp64) or float (fp32).
// rows [f0, f1) of [0, m] (row m = the property)
void launch_gather(const double* values, const double* y, const int64_t* perm, int64_t m, int64_t s,
                   int precision, void* Xp, void* yp, int64_t f0, int64_t f1, cudaStream_t st);
// Per (feature, task): center, normalize, write Z rows (features 0..m-1 unit-norm
// centered, row m = centered y), plus q = |x_c|^2/|x|^2 and |x|^2 per (task, feature)
// and |y|^2 per task.
// Ozaki digit planes written by the normalize kernel (Q == nullptr: none)
constexpr int OZ_DIGITS = 4;
struct DigitOut {
    int8_t* Q;             // [OZ_DIGITS][R][KP]
    int64_t R, KP;
    const int64_t* koff;   // (T+1,) device: task segment offsets in K (multiples of 64)
    int* ex;               // [T][R] row exponents
    bool write_z = true;   // also write the fp64 rows Z (only the DMMA Gram reads them)
    double* musc = nullptr;  // [T][R][2] the rows' (mean, scale): z = (x - mean) * scale (k_oz_fixup)
};
void launch_normalize(const void* Xp, const void* yp, int precision, int64_t m, int64_t s,
                      const int64_t* bounds_d, const int64_t* zoff_d, int T, int64_t sp, double* Z,
                      double* qf, double* un2, double* yyu, int64_t f0, int64_t f1, DigitOut dig, cudaStream_t st);

// gather + normalize fused (stage.cu k_stage_rows) when a task segment fits in shared memory
// (max_rows rows), else the two kernels above
bool stage_rows_fused(int64_t max_rows, const DigitOut& dig);
void launch_stage_rows(const double* values, const double* y, const int64_t* perm, int64_t m, int64_t s, int precision,
                       void* Xp, void* yp, const int64_t* bounds_d, const int64_t* zoff_d, int T, int64_t sp,
                       double* Z, double* qf, double* un2, double* yyu, int64_t f0, int64_t f1, DigitOut dig,
                       int64_t max_rows, cudaStream_t st);

// Residuals of `count` models (models.residuals / predict, models.py:44-83): out[c][i] =
// y[i] - (coef[c][t][n] + sum_k coef[c][t][k] * values[tup[c][k]][i]) for sample i of task t,
// numpy's operation order (explicit roundings), in the caller's sample order.
void launch_residuals(const double* values, const double* y, const int64_t* perm, const int64_t* bounds, int T,
                      int64_t s, int n, const int64_t* tup, const double* coef, int64_t count, double* out,
                      cudaStream_t st);

// rho, dead, rho_cap, iforce from qf / un2 (stage.cu), and NaN rows/cols of dead features in G
void launch_feature_flags(double tol, int fp32, const double* qf, const double* un2, const double* rows, int64_t m, int64_t mp, int T,
                          double* umin, double* rho, double* rho_cap, unsigned char* dead, unsigned char* iforce,
                          double* G, const double* yyu, double* ynorm, cudaStream_t st);

// ---- Gram (gram.cu): G[t] = Z_t Z_t^T on DMMA, (mp x mp) per task ----
// The T x (upper-triangle 64 x 64 blocks) are numbered linearly; nshards == 1 computes all of
// them into G, otherwise shard `shard` computes its contiguous range of gram_shard_blocks()
// into `pack` (row-major 64 x 64 tiles), exchanged by an all-gather and scattered by
// launch_gram_unpack (recv = nshards x per-shard tiles, in shard order).
int64_t gram_blocks(int64_t mp, int T);
int64_t gram_shard_blocks(int64_t mp, int T, int nshards);
void launch_gram(const double* Z, int64_t sp, const int64_t* zoff_d, int T, int64_t mp, double* G, int shard,
                 int nshards, double* pack, cudaStream_t st);
void launch_gram_unpack(const double* recv, int T, int64_t mp, double* G, cudaStream_t st);
// Blocks of every task whose column block-row bb lies in [B0, B1) (bb >= ba): the part of the
// Gram that becomes computable once Z's block-rows < B1 are staged (overlapped stage).
void launch_gram_cols(const double* Z, int64_t sp, const int64_t* zoff_d, int T, int64_t mp, double* G, int B0,
                      int B1, cudaStream_t st);
// diagonal of the feature rows := 1 (unit-norm columns; NaN rows stay NaN)
void launch_unit_diag(double* G, int T, int64_t m, int64_t mp, cudaStream_t st);
// Features the reference's rank rule rejects in every tuple: NaN their Gram row and column (all tasks).
void launch_mark_dead(double* G, const int32_t* dead, int ndead, int T, int64_t mp, cudaStream_t st);

// ---- Gram on the INT8 tensor cores by Ozaki splitting (ozaki.cu) ----
struct OzFix {
    int* rows;      // (cap,) loose rows (device)
    int* count;     // loose rows found (device, may exceed cap)
    int cap;
    unsigned char* flags;  // (m + 1,) device scratch: the rows' loose flags
};
int64_t ozaki_q_bytes(int64_t mp, int T, const int64_t* rpad_h, int64_t* KP_out);
// digits_ready: the normalize kernel already wrote Q / ex (and koff_d); otherwise split Z here
int launch_ozaki_gram(const double* Z, int64_t sp, const int64_t* zoff_d, const int64_t* rpad_h, int T, int64_t m,
                      int64_t mp, const double* rows_d, double* G, double* eta_d, int8_t* Q, int* ex, int64_t* koff_d,
                      bool digits_ready, cudaStream_t st, const OzFix* fix = nullptr);
// pieces of the same, for the overlapped stage: tiles of the column blocks [gb0, gb1) (64 wide)
// and the error-bound kernel (after all tiles)
int ozaki_col_blocks(int64_t mp);
int ozaki_blocks_ready(int64_t r1);  // column blocks complete once rows < r1 have landed
int launch_ozaki_tiles(int T, int64_t mp, const int64_t* rpad_h, const int8_t* Q, const int* ex,
                       const int64_t* koff_d, double* G, int gb0, int gb1, cudaStream_t st);
// eta_t (see ozaki.cu).  fix != nullptr: rows whose own error term exceeds OZ_ETA_MAX in some task
// are listed in fix->rows (count in fix->count, at most fix->cap listed) and left out of eta_t:
// launch_ozaki_fixup recomputes their Gram rows in fp64
constexpr double OZ_ETA_MAX = 1e-6;  // the screen's limit on eta_t (larger: DMMA Gram)
void launch_ozaki_eta(int T, int64_t m, int64_t mp, const int* ex, const double* rows_d, const double* G, double* eta_d,
                      cudaStream_t st, const OzFix* fix = nullptr);
// fp64 Gram rows and columns of the listed loose rows from Xp / yp and the stored (mean, scale)
// (every task; a no-op when the count is 0 or above cap -- the host then takes the DMMA Gram)
void launch_ozaki_fixup(const void* Xp, const void* yp, int precision, int64_t m, int64_t s, const int64_t* bounds_d,
                        int T, const double* musc, int64_t R, int64_t mp, const OzFix& fix, double* G, cudaStream_t st);
// Q / ex zero fill of the rows the normalize kernel does not write (m+1 .. R-1) and koff upload
void ozaki_prepare_digits(int64_t m, int64_t mp, int T, const int64_t* rpad_h, int8_t* Q, int* ex, int64_t* koff_d,
                          DigitOut* out, cudaStream_t st, double* musc = nullptr);

// ---- bit-exact Householder (exact.cu) ----
struct ExactArgs {
    const void* Xp;         // (m, s) working dtype, permuted
    const void* yp;         // (s,)
    const int64_t* bounds;  // (T+1,) device
    int T;
    int64_t m, s;
    int n;
    double tol;
    int precision;
    // tuple source: explicit tuples (count x n) or ranks (count)
    const int64_t* tuples;
    const int64_t* ranks;
    const int64_t* binom;  // (n+1) x (m+1) table, C(a,k) at [k*(m+1)+a]
    int64_t count;
    // outputs (per tuple)
    int32_t* ok;      // (count,)
    double* score;    // (count,) sum_t ssr / s, +inf when deficient
    double* coef;     // (count, T, n+1) or nullptr
    double* ssr;      // (count, T) or nullptr
    void* scratch;    // interleaved scratch
    int64_t scratch_threads;
    int64_t ld;       // max rows over tasks
};
// Runs in chunks of args.scratch_threads threads (one per (tuple, task)).
void launch_exact(const ExactArgs& a, double* ssr_tmp, int32_t* ok_tmp, cudaStream_t st, int64_t* launches);

// ---- QR screen for uncertifiable tuples (qr.cu) ----
struct QrArgs {
    const double* Xp;       // (m, s) fp64, permuted
    const double* yp;
    const int64_t* bounds;  // (T+1,) device
    int T;
    int64_t m, s;
    int n;
    const int64_t* ranks;   // (count,)
    const int64_t* binom;
    double* ssr;            // (count*T) scratch
    double* ratio;          // (count*T) scratch
    double* score;          // (count,) sum_t ssr / s
    double* min_ratio;      // (count,) min over tasks of min|R_jj| / max|R_jj|
    int64_t g0, total;      // set by the launcher
};
void launch_qr_screen(const QrArgs& a, int64_t count, cudaStream_t st, int64_t* launches);
// the same screen through a double-double Gram of every staged column (ddgram.cu): Hhi / Hlo
// (T x LD x LD each, LD = dd_gram_ld(m)) are filled unless gram_ready
void launch_qr_finalize(const QrArgs& a, int64_t count, cudaStream_t st, int64_t* launches);  // score, min_ratio
int64_t dd_gram_ld(int64_t m);
int64_t dd_gram_lo_doubles(int64_t m, int T);
bool dd_screen_pays(int64_t nill, int n, int T, int64_t m, int64_t s);
void launch_dd_screen(const QrArgs& a, int64_t count, double* Hhi, double* Hlo, bool gram_ready, cudaStream_t st,
                      int64_t* launches);
// ranks of the screened ill tuples that may still reach the top list (selection on the device)
void launch_qr_select(const double* score, const double* min_ratio, const int64_t* ranks, int64_t count, double tol,
                      double sk, double yy_s, int64_t* sel, unsigned long long* nsel, int64_t cap, cudaStream_t st);

// ---- screened fit (fit3.cu) ----
// global lower-bound histogram behind the shared threshold (fitcommon.cuh): HIST_SUB sub-bins
// per binary exponent, HIST_EXP exponents below the top (the total |y|^2)
constexpr int HIST_SUB_BITS = 5;
constexpr int HIST_EXP = 44;
constexpr int HIST_BINS = HIST_EXP << HIST_SUB_BITS;
inline int hist_base_for(double top) {
    unsigned long long u;
    __builtin_memcpy(&u, &top, 8);
    const int e = (int)((u >> 52) & 0x7ff);
    return (e + 1 - HIST_EXP) << HIST_SUB_BITS;
}
// TMA descriptors for the Gram viewed as a 2-D (T*mp rows x mp columns) f64 tensor;
// one per box shape the kernel stages (built by the launcher, which knows the tile shape).
struct alignas(64) TmaDesc {
    unsigned long long opaque[16];
};
// per-thread error message of the C ABI (api.cu): returns `code`
int set_error(int code, const char* msg);

// ---- streamed last rung: value dedup on the device (dedup.cu) ----
struct DedupTable {
    unsigned long long* lo;     // [mask + 1] fingerprint words
    unsigned long long* hi;
    unsigned long long* owner;  // (epoch << 32) | index of the first occurrence
    unsigned* state;            // 0 empty, 1 being written, 2 ready
    unsigned long long* used;   // entries inserted
    unsigned long long mask;    // capacity - 1 (a power of two)
};
void launch_dedup_insert(DedupTable t, const unsigned char* valid, const unsigned long long* hash, int64_t count,
                         unsigned long long epoch, cudaStream_t st);
void launch_dedup_mark(DedupTable t, const unsigned char* valid, const unsigned long long* hash, int64_t count,
                       unsigned long long epoch, unsigned char* kept, cudaStream_t st);
void launch_dedup_rehash(DedupTable from, DedupTable to, cudaStream_t st);

// ---- host -> device copies from pageable memory (hostcopy.cu) ----
struct HostStager;
HostStager* host_stager_create();  // nullptr when no pinned memory could be had
void host_stager_destroy(HostStager* h);
bool host_is_pinned(const void* p);
cudaError_t host_stager_copy_rows(HostStager* h, void* dst, const std::function<const void*(int64_t)>& row,
                                  int64_t nrows, size_t row_bytes, cudaStream_t st);

constexpr int kSeedW = 5;  // int64 slots per threshold-seed subset (n <= 5)
struct FitArgs {
    TmaDesc tmJ;  // box: 32 columns (j-block) x IB rows
    TmaDesc tmK;  // box: KSPAN columns (k- or l-span) x IB rows
    TmaDesc tmC;  // box: 2 columns (one Gram column + its neighbour) x IB rows
    TmaDesc tmH;  // box: 32 columns (j-block) x KSPAN rows (the unit's hoist block C[k-span, j-block])
    const double* G;         // [T][mp][mp] normalized Gram, y at index m
    const double* qf;        // [T][m]
    const double* un2;       // [T][m]
    const double* rowsd;     // [T] rows per task as double
    const double* eta;       // [T] per-entry Gram error bound
    const double* rho;       // [T][m] 1/sqrt(q): uncentered / centered norm ratio per feature
    const double* rho_cap;   // [T] rho assumed for the sweep feature i unless it is flagged in iforce
    const double* ynorm;     // [T] |y_t| (uncentered)
    const unsigned char* iforce;  // [m] 1 = rho_i exceeds rho_cap: tuples with this i take the slow path
    int n;                   // tuple dimension (for the reference's backward-error constant)
    const int64_t* binom;    // (n+1) x (m+1)
    const int4* units;       // unit table
    int n_units;
    int* unit_counter;
    int64_t m, mp;
    int T;
    int64_t N_total;         // C(m, n)
    int64_t rank_lo, rank_hi;
    int ranged;
    double tol2;             // reference rank rule: tol^2
    int ref_fp32;            // the reference computes in float32 (precision="fp32"): its rounding model
    // candidate state
    int kc;                  // per-warp keep K'
    int collect;             // 0 = per-warp top-K' lists; 1 = collect every lb < theta0 into coll_*;
                             // 2 = collect below the histogram threshold (large keep, K' = kc)
    double theta0;
    unsigned long long* theta_g;
    unsigned* hist;          // [HIST_BINS] global lower-bound histogram (fitcommon.cuh)
    int64_t* seed_tup;       // [SEED_MAX][kSeedW] threshold-seed subsets (fitcommon.cuh)
    double* seed_ub;         // [SEED_MAX] their upper bounds
    int* seed_n;             // subset count
    double* seed_cap;        // out: the keep-th smallest certified upper bound of the seed (SSR units)
    int keep;                // models kept (search parts: the seed caps the global keep-th score)
    int hist_base;           // bin offset: (biased exponent of the top) - HIST_EXP, times HIST_SUB
    double* wl_lb;           // [n_warp_slots][kc]
    int64_t* wl_rank;
    int* wl_cnt;             // [n_warp_slots]
    int64_t* ill;            // ill-conditioned tuple ranks
    unsigned long long* ill_cnt;
    int64_t ill_cap;
    double* coll_lb;
    int64_t* coll_rank;
    unsigned long long* coll_cnt;
    int64_t coll_cap;
    unsigned long long* n_eval;  // out (optional): task-tuple evaluations of the sweep (executed work)
    // (optional, n = 3) row-block maxima of the first task slot's Gram for the tile screen, blocks
    // of the sweep's tile height: [col <= m][block] max |C[i, col]| (col = m: max |c_i|; +inf for a
    // flagged or NaN row), [j-block][block], then the slot's task index (fit3.cu: k_tile_max)
    double* tmax = nullptr;
    unsigned long long* n_screen = nullptr;  // out (optional): tile-screen tests (warp-level)
};
// doubles fit3_launch needs in FitArgs::tmax for an m-feature problem
int64_t fit3_tmax_doubles(int64_t m, int64_t mp);
// n = 1 (fit1.cu): dense lower bounds of the features [rb, re) (+inf: ill or dead; ill ranks appended)
void launch_fit1(const FitArgs& a, int64_t rb, int64_t re, double* out_lb, int64_t* out_rank, cudaStream_t st);
int fit3_launch(const FitArgs& a, int nsm, cudaStream_t st);  // returns grid size (warp slots / 8)
int fit3_grid(int T, int nsm);                                // grid fit3_launch will use
int fit3_max_tasks();
int fit_slots_per_cta();   // warp candidate slots per CTA (n = 2, 4)
int fit3_slots_per_cta(int T);  // the same for the n = 3 sweep (T tasks)
int fit3_kspan(int T);
std::vector<int4> fit3_units(int64_t m, int T, int64_t N_total, const std::vector<int64_t>& c2_prefix,
                             int64_t rank_lo, int64_t rank_hi, bool tunable = true);
// lower bound + flags for explicit 3-tuples (same arithmetic as the fit kernel's slow path)
void launch_screen3(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st);

// ---- screened fit, n = 2 (fit2.cu) ----
int fit2_launch(const FitArgs& a, int nsm, cudaStream_t st);
int fit2_grid(int T, int nsm);
std::vector<int4> fit2_units(int64_t m, const std::vector<int64_t>& c1_prefix, int64_t rank_lo, int64_t rank_hi);
void launch_screen2(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st);

// ---- screened fit, n = 4 (fit4.cu) ----
int fit4_launch(const FitArgs& a, int nsm, cudaStream_t st);
int fit4_grid(int T, int nsm);
std::vector<int4> fit4_units(int64_t m, int T, const std::vector<int64_t>& c3_prefix, int64_t rank_lo,
                             int64_t rank_hi);
// ---- screened fit, n = 5 (fit5.cu) ----
int fit5_launch(const FitArgs& a, int nsm, cudaStream_t st);
int fit5_grid(int T, int nsm);
std::vector<int4> fit5_units(int64_t m, int T, const std::vector<int64_t>& c4_prefix, int64_t rank_lo,
                             int64_t rank_hi);
void launch_screen5(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st);
void launch_screen4(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st);

// 3-D int8 tensor (x = cols contiguous, y = rows, z = planes), box (bx, by, 1), 64-byte swizzle
bool make_tma_i8_3d(TmaDesc* out, const void* base, unsigned long long cols, unsigned long long rows,
                    unsigned long long planes, unsigned bx, unsigned by);
// Encode a 2-D f64 tiled TMA descriptor over G ([rows x cols], row stride = cols) with box (bx, by).
bool make_tma_2d(TmaDesc* out, const double* G, unsigned long long cols, unsigned long long rows, unsigned bx,
                 unsigned by);

// ---- candidate gather (merge.cu) ----
void launch_gather_candidates(const double* wl_lb, const int64_t* wl_rank, const int* wl_cnt, int slots,
                              int kc, const unsigned long long* theta_g, double* out_lb,
                              int64_t* out_rank, unsigned long long* out_cnt, cudaStream_t st);
// sort (lb, rank) pairs ascending by (lb, rank) in place (sort.cu: shared-memory bitonic blocks
// + merge-path rounds); returns the number of launches (-1: temp too small)
size_t sort_pairs_temp_bytes(int64_t n);
int sort_pairs(double* lb, int64_t* rank, double* lb_tmp, int64_t* rank_tmp, int64_t n, void* temp,
               size_t temp_bytes, cudaStream_t st);

// ---- SIS projection scores (sis.cu), bit-identical to screening._chunk_scores ----
int sis_max_targets();
void launch_sis_targets(const double* y, int R, int64_t s, const int64_t* perm, const int64_t* bounds, int T,
                        double* yc, double* sy, cudaStream_t st);
// dest[j]: shared-memory slot of raw sample j (task t's segment at tpoff[t], lane stride
// tE[t] + 1 with tE[t] = max(1, pow2ceil(n_t) / 32)); rowlen = the padded row length
int launch_sis_scores(const double* F, int64_t k, int64_t s, const int64_t* perm, const int* dest,
                      const int64_t* bounds, const int* tE, const int* tpoff, int rowlen, int T, const double* yc,
                      const double* sy, int R, double* out, int nsm, cudaStream_t st);

// ---- final-rung candidates (gen.cu): values, validity, fingerprints ----
enum GenKind {
    GEN_COPY = 0,  // the row itself (the pool's own fingerprints)
    GEN_ADD = 1,
    GEN_SUB = 2,
    GEN_MUL = 3,
    GEN_DIV = 4,
    GEN_ABS_DIFF = 5,
    GEN_SQRT = 6,
    GEN_SQ = 7,
    GEN_CB = 8,
    GEN_INV = 9,
    GEN_ABS = 10,
    GEN_VALUES = 11,  // precomputed candidate rows (libm operators)
};
void launch_gen_eval(const void* A, int fp32, int64_t s, const int* pi, const int* pj, int count, int kind, double tol,
                     double min_abs, double max_abs, double dedup_tol, double* vals, unsigned char* valid,
                     unsigned long long* hash, cudaStream_t st);
void launch_gen_gather(const double* vals, int64_t s, const int* rows, int count, int fp32, void* out,
                       cudaStream_t st);

// ---- misc ----
double fp64_peak_tflops(int dev);

}  // namespace l0s
