// api.cu -- the C ABI (include/l0search.h): context, staging, search orchestration.
//
// Search = screened fit kernel over every tuple (fit3.cu) -> device merge of
// the per-warp top-K' lists (merge.cu) -> bit-exact Householder refit of the
// candidates and of every tuple the screen could not certify (exact.cu) ->
// (score, rank) order, certification, optional threshold rescan.  See
// DESIGN.md for the proof obligations behind "certified".
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/l0search.h"
#include "common.cuh"
#include "kernels.h"

using namespace l0s;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) return fail(L0S_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, bytes < 256 ? 256 : bytes);
        if (e == cudaSuccess) n = bytes < 256 ? 256 : bytes;
        return e;
    }
    // grow to `bytes` keeping the first `keep` bytes (device copy on `st`)
    cudaError_t grow(size_t bytes, size_t keep, cudaStream_t st) {
        if (bytes <= n && p) return cudaSuccess;
        void* q = nullptr;
        const size_t cap = bytes + bytes / 4;
        cudaError_t e = cudaMalloc(&q, cap);
        if (e != cudaSuccess) return e;
        if (p && keep) {
            e = cudaMemcpyAsync(q, p, keep, cudaMemcpyDeviceToDevice, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) {
                cudaFree(q);
                return e;
            }
        }
        if (p) cudaFree(p);
        p = q;
        n = cap;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <typename T>
    T* as() const {
        return (T*)p;
    }
};

// C(a, b) with 128-bit intermediates, saturated at INT64_MAX
int64_t binom_sat(int64_t a, int64_t b) {
    if (b < 0 || a < 0 || b > a) return 0;
    if (b > a - b) b = a - b;
    unsigned __int128 r = 1;
    for (int64_t i = 1; i <= b; ++i) {
        r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
        if (r > (unsigned __int128)INT64_MAX) return INT64_MAX;
    }
    return (int64_t)r;
}

struct Rec {  // bit-exact record of one refit tuple
    double score;
    std::vector<double> coef, ssr;
};

}  // namespace

struct l0s_ctx {
    int dev = 0, nsm = 0;
    cudaStream_t st = nullptr;
    cudaStream_t cst = nullptr;  // H2D copies of the overlapped stage
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    static constexpr int kChunks = 8;
    cudaEvent_t cev[kChunks + 1] = {};
    cudaEvent_t sev[5] = {};         // unchunked stage: gather | normalize | (Gram: ev[2..3]) | flags
    bool stage_timed = false;
    bool stage_fused = false;  // the timed staging pass was k_stage_rows (gather + normalize in one)
    // staged problem
    bool staged = false;
    int64_t m = 0, s = 0, mp = 0, sp = 0, ld = 0;
    int T = 0, prec = 0;
    std::vector<int64_t> bounds_h, zoff_h, rpad_h;
    std::vector<double> rows_h, eta_h, yyu_h;
    double ms_gram = 0.0;
    double ms_gram_k = 0.0;  // the Gram kernel alone (unchunked stage)
    DBuf in_values, in_y, in_perm, bounds_d, zoff_d, Xp, yp, Z, G, qf, un2, yyu, rowsd, eta_d;
    DBuf rho, rho_cap, ynorm, iforce, dead, umin, tmax;
    int64_t n_dead = 0, n_iforce = 0;
    bool shard_pending = false;  // l0s_stage_shard done, l0s_stage_finish due
    bool host_staged = false;    // in_values / in_y / in_perm hold the staged problem's inputs
    bool gram_timed = false;     // ev[2..3] bracket the Gram kernel of this stage
    int gram_mode = 0;           // L0S_GRAM_AUTO / _DMMA / _OZAKI (l0s_set_gram_mode)
    bool gram_ozaki = false;     // the staged Gram came from the INT8 path (eta on the device)
    bool digits_ready = false;   // the normalize kernel wrote the Ozaki digits of this stage
    DBuf oz_q, oz_ex, oz_koff;
    // loose rows of the INT8 Gram (a row's own error term above OZ_ETA_MAX) recomputed in fp64:
    // oz_musc = the rows' (mean, scale) beside their digits, oz_fix = (kFixCap rows, count)
    static constexpr int kFixCap = 64;
    DBuf oz_musc, oz_fix;
    bool fix_on = false;  // this stage's eta left the listed rows out; k_oz_fixup is due
    int fix_count = 0;    // loose rows of the last stage (l0s_stage_info)
    // binomial table (k <= binom_n) x (a <= m)
    DBuf binom;
    int binom_n = -1;
    int64_t binom_m = -1;
    // search workspace
    DBuf units, ucount, n_eval, theta_g, hist, seedbuf, wl_lb, wl_rank, wl_cnt, ill, ill_cnt, cand_lb, cand_rank, cand_cnt, sort_tmp,
        lb_tmp, rank_tmp, coll_lb, coll_rank, coll_cnt;
    DBuf ex_scratch, ex_ssr_tmp, ex_ok_tmp, ex_ok, ex_score, ex_coef, ex_ssr, ex_ranks, ex_tuples;
    DBuf qr_ssr, qr_ratio, qr_score, qr_minr;
    DBuf ddg_hi, ddg_lo;     // double-double Gram of the staged columns (ddgram.cu), on first use
    bool ddg_ready = false;  // ... for the current stage
    // SIS projection scores
    DBuf sis_y, sis_yc, sis_sy, sis_perm, sis_bounds, sis_F, sis_out, sis_dest, sis_tE, sis_tpoff;
    // final-rung candidates (gen.cu)
    DBuf gen_pool, gen_pi, gen_pj, gen_vals, gen_valid, gen_hash, gen_take, gen_rows, gen_out;
    int64_t gen_n = 0, gen_s = 0, gen_count = 0, gen_taken = 0;
    int gen_fp32 = 0;
    int sis_R = 0, sis_T = 0, sis_rowlen = 0;
    int64_t sis_s = 0;
    std::unordered_map<int64_t, Rec> recs;  // records of this search's refit candidates
    std::vector<int4> units_h;
    int64_t units_key[7] = {-1, -1, -1, -1, -1, -1, -1};
    int part = 0, nparts = 1;  // l0s_search_part: this context screens units u with u % nparts == part
    l0s_exchange_fn exch = nullptr;  // l0s_set_part_exchange
    void* exch_user = nullptr;
    bool exch_pending = false;  // this l0s_search_part call has not exchanged yet
    HostStager* stager = nullptr;  // pinned ring for pageable host inputs (hostcopy.cu), on first use
    const double* src_values = nullptr;  // the staged inputs, caller's sample order (device)
    const double* src_y = nullptr;
    const int64_t* src_perm = nullptr;
    DBuf res_tup, res_coef, res_out;
    DBuf dd_lo, dd_hi, dd_owner, dd_state, dd_used, dd_kept, dd_seed;  // last-rung value dedup (dedup.cu)
    unsigned long long dd_mask = 0, dd_epoch = 0;

    ~l0s_ctx() {
        if (stager) host_stager_destroy(stager);
        DBuf* all[] = {&in_values, &in_y, &in_perm, &bounds_d, &zoff_d, &Xp, &yp, &Z, &G, &qf, &un2, &yyu, &rowsd,
                       &eta_d, &rho, &rho_cap, &ynorm, &iforce, &dead, &umin, &tmax, &binom, &units, &ucount, &n_eval, &theta_g, &hist, &seedbuf, &wl_lb, &wl_rank, &wl_cnt, &ill, &ill_cnt,
                       &cand_lb, &cand_rank, &cand_cnt, &sort_tmp, &lb_tmp, &rank_tmp, &coll_lb, &coll_rank,
                       &coll_cnt, &ex_scratch, &ex_ssr_tmp, &ex_ok_tmp, &ex_ok, &ex_score, &ex_coef, &ex_ssr,
                       &ex_ranks, &ex_tuples, &qr_ssr, &qr_ratio, &qr_score, &qr_minr, &ddg_hi, &ddg_lo, &sis_y, &sis_yc, &sis_sy, &sis_perm,
                       &sis_bounds, &sis_F, &sis_out, &sis_dest, &sis_tE, &sis_tpoff, &oz_q, &oz_ex, &oz_koff, &oz_musc, &oz_fix,
                       &res_tup, &res_coef, &res_out, &dd_lo, &dd_hi, &dd_owner, &dd_state, &dd_used, &dd_kept, &dd_seed, &gen_pool, &gen_pi, &gen_pj, &gen_vals, &gen_valid, &gen_hash, &gen_take, &gen_rows, &gen_out};
        for (DBuf* b : all) b->release();
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : cev)
            if (e) cudaEventDestroy(e);
        for (auto& e : sev)
            if (e) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
        if (cst) cudaStreamDestroy(cst);
    }
};

namespace {

int ensure_binom(l0s_ctx* c, int n) {
    int need = std::max(n, 3);
    if (c->binom_n >= need && c->binom_m == c->m) return L0S_OK;
    std::vector<int64_t> tab((size_t)(need + 1) * (size_t)(c->m + 1));
    for (int k = 0; k <= need; ++k)
        for (int64_t a = 0; a <= c->m; ++a) tab[(size_t)k * (c->m + 1) + a] = binom_sat(a, k);
    CK(c->binom.ensure(tab.size() * sizeof(int64_t)));
    CK(cudaMemcpyAsync(c->binom.p, tab.data(), tab.size() * sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    c->binom_n = need;
    c->binom_m = c->m;
    return L0S_OK;
}

struct ExactOut {
    std::vector<int32_t> ok;
    std::vector<double> score;
};

// Bit-exact scores (and optionally coef/ssr) for `count` tuples given by device ranks or device tuples.
int run_exact(l0s_ctx* c, int n, const int64_t* ranks_d, const int64_t* tuples_d, int64_t count, bool want_coef,
              int64_t* launches) {
    const int p = n + 1;
    size_t wsz = c->prec == L0S_PREC_FP32 ? 4 : 8;
    // scratch budget: <= 1 GiB of interleaved systems
    int64_t per_sys = (int64_t)(p + 1) * std::max<int64_t>(c->ld, 1) * (int64_t)wsz;
    int64_t budget = (int64_t)1 << 30;
    int64_t cap_thr = std::max<int64_t>(c->T, std::min<int64_t>(budget / per_sys, count * c->T));
    cap_thr = std::max<int64_t>(cap_thr, 1);
    // systems that fit in shared memory never touch the interleaved scratch (exact.cu)
    const bool smem_path = per_sys <= (int64_t)200 * 1024 && n <= 15;
    if (!smem_path) CK(c->ex_scratch.ensure((size_t)(cap_thr * per_sys)));
    CK(c->ex_ssr_tmp.ensure(sizeof(double) * (size_t)std::max<int64_t>(count * c->T, 1)));
    CK(c->ex_ok_tmp.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(count * c->T, 1)));
    CK(c->ex_ok.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(count, 1)));
    CK(c->ex_score.ensure(sizeof(double) * (size_t)std::max<int64_t>(count, 1)));
    CK(c->ex_ssr.ensure(sizeof(double) * (size_t)std::max<int64_t>(count * c->T, 1)));
    if (want_coef) CK(c->ex_coef.ensure(sizeof(double) * (size_t)std::max<int64_t>(count * c->T * p, 1)));
    ExactArgs a{};
    a.Xp = c->Xp.p;
    a.yp = c->yp.p;
    a.bounds = c->bounds_d.as<int64_t>();
    a.T = c->T;
    a.m = c->m;
    a.s = c->s;
    a.n = n;
    a.tol = c->prec == L0S_PREC_FP32 ? 1e-5 : 1e-10;  // RANK_TOL_FACTOR, lsq.py:23
    a.precision = c->prec;
    a.tuples = tuples_d;
    a.ranks = ranks_d;
    a.binom = c->binom.as<int64_t>();
    a.count = count;
    a.ok = c->ex_ok.as<int32_t>();
    a.score = c->ex_score.as<double>();
    a.coef = want_coef ? c->ex_coef.as<double>() : nullptr;
    a.ssr = c->ex_ssr.as<double>();
    a.scratch = c->ex_scratch.p;
    a.scratch_threads = cap_thr;
    a.ld = std::max<int64_t>(c->ld, 1);
    launch_exact(a, c->ex_ssr_tmp.as<double>(), c->ex_ok_tmp.as<int32_t>(), c->st, launches);
    CK(cudaGetLastError());
    return L0S_OK;
}

// CTAs assumed when splitting units into search parts (a B200's 148 SMs, one CTA each)
constexpr int kPartGridCtas = 148;

// keep above which the screened path collects candidates globally instead of per-warp lists,
// and the largest keep it takes (K' = keep + 32 candidates refit exactly)
constexpr int64_t kKeepLists = 96;
constexpr int64_t kKeepMax = 4064;

struct Cand {
    double score;
    int64_t rank;
};
bool cand_less(const Cand& x, const Cand& y) { return x.score < y.score || (x.score == y.score && x.rank < y.rank); }

__global__ void k_iota(int64_t* out, int64_t start, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = start + i;
}

// keep the best `keep` finite (score, rank) in `best` (sorted)
void merge_best(std::vector<Cand>& best, const std::vector<Cand>& more, int64_t keep) {
    for (const Cand& x : more)
        if (std::isfinite(x.score)) best.push_back(x);
    std::sort(best.begin(), best.end(), cand_less);
    best.erase(std::unique(best.begin(), best.end(),
                           [](const Cand& x, const Cand& y) { return x.rank == y.rank; }),
               best.end());
    if ((int64_t)best.size() > keep) best.resize((size_t)keep);
}

// Exact scores for device ranks [0, count) of c->ex_ranks; appends finite (score, rank) to out.
// Exact scores for `count` device ranks; with `recs`, also keep each tuple's coefficients and
// per-task ssr (small candidate sets), so the final records need no second launch.
// The exact refit of `count` ranks on the device, split so a caller can queue more work (and
// host copies) between the launch and the collection: exact_launch queues the kernels and the
// result copies into `pend`, exact_collect waits and appends (score, rank) to `out`.
struct ExactPending {
    int64_t count = 0;
    bool keep_rec = false;
    std::vector<double> sc, cf, ss;
    std::vector<int64_t> rk;
};

int exact_launch(l0s_ctx* c, int n, const int64_t* ranks_d, int64_t count, ExactPending& pend, int64_t* launches,
                 bool want_rec) {
    pend.count = count;
    if (count <= 0) return L0S_OK;
    pend.keep_rec = want_rec && count <= 4096;
    int rc = run_exact(c, n, ranks_d, nullptr, count, pend.keep_rec, launches);
    if (rc) return rc;
    const int p = n + 1;
    pend.sc.resize((size_t)count);
    pend.rk.resize((size_t)count);
    CK(cudaMemcpyAsync(pend.sc.data(), c->ex_score.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(pend.rk.data(), ranks_d, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, c->st));
    if (pend.keep_rec) {
        pend.cf.resize((size_t)(count * c->T * p));
        pend.ss.resize((size_t)(count * c->T));
        CK(cudaMemcpyAsync(pend.cf.data(), c->ex_coef.p, sizeof(double) * pend.cf.size(), cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(pend.ss.data(), c->ex_ssr.p, sizeof(double) * pend.ss.size(), cudaMemcpyDeviceToHost, c->st));
    }
    return L0S_OK;
}

int exact_collect(l0s_ctx* c, int n, ExactPending& pend, std::vector<Cand>& out,
                  std::unordered_map<int64_t, Rec>* recs) {
    if (pend.count <= 0) return L0S_OK;
    CK(cudaStreamSynchronize(c->st));
    const int p = n + 1;
    for (int64_t i = 0; i < pend.count; ++i) {
        out.push_back({pend.sc[(size_t)i], pend.rk[(size_t)i]});
        if (pend.keep_rec && recs && std::isfinite(pend.sc[(size_t)i])) {
            Rec& r = (*recs)[pend.rk[(size_t)i]];
            r.score = pend.sc[(size_t)i];
            r.coef.assign(pend.cf.begin() + i * c->T * p, pend.cf.begin() + (i + 1) * c->T * p);
            r.ssr.assign(pend.ss.begin() + i * c->T, pend.ss.begin() + (i + 1) * c->T);
        }
    }
    pend.count = 0;
    return L0S_OK;
}

int exact_ranks_to_host(l0s_ctx* c, int n, const int64_t* ranks_d, int64_t count, std::vector<Cand>& out,
                        int64_t* launches, std::unordered_map<int64_t, Rec>* recs = nullptr) {
    ExactPending pend;
    int rc = exact_launch(c, n, ranks_d, count, pend, launches, recs != nullptr);
    if (rc) return rc;
    return exact_collect(c, n, pend, out, recs);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

namespace l0s {
int set_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace l0s

extern "C" {

const char* l0s_last_error(void) { return g_err.c_str(); }
int l0s_version(void) { return 1; }

int l0s_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *count = n;
    return L0S_OK;
}

int l0s_create(int device, l0s_ctx** out) {
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(L0S_ENODEV, "no CUDA device visible");
    if (device < 0 || device >= n) return fail(L0S_EINVAL, "device %d out of range [0, %d)", device, n);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(L0S_ENODEV, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
    CK(cudaSetDevice(device));
    l0s_ctx* c = new l0s_ctx();
    c->dev = device;
    c->nsm = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return fail(L0S_ECUDA, "stream creation failed");
    }
    if (cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess) {
        cudaStreamDestroy(c->st);
        delete c;
        return fail(L0S_ECUDA, "stream creation failed");
    }
    for (auto& e : c->ev) cudaEventCreate(&e);
    for (auto& e : c->cev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (auto& e : c->sev) cudaEventCreate(&e);
    if (const char* g = getenv("L0S_GRAM_MODE"))  // experiments: auto | dmma | ozaki
        c->gram_mode = !strcmp(g, "dmma") ? L0S_GRAM_DMMA : (!strcmp(g, "ozaki") ? L0S_GRAM_OZAKI : L0S_GRAM_AUTO);
    *out = c;
    return L0S_OK;
}

int l0s_destroy(l0s_ctx* c) {
    if (!c) return L0S_OK;
    cudaSetDevice(c->dev);
    cudaStreamSynchronize(c->st);
    delete c;
    return L0S_OK;
}

// stage up to (not including) the Gram: validation, layout, H2D, gather + normalize into Z
static int stage_prepare(l0s_ctx* c, const double* values, int64_t m, int64_t s, const double* y, const int64_t* perm,
                         const int64_t* bounds, int ntasks, int precision, int is_device) {
    if (!c) return fail(L0S_EINVAL, "null context");
    if (m < 1 || s < 1 || ntasks < 1) return fail(L0S_EINVAL, "need m >= 1, s >= 1, ntasks >= 1 (got %lld, %lld, %d)", (long long)m, (long long)s, ntasks);
    if (precision != L0S_PREC_FP64 && precision != L0S_PREC_FP32) return fail(L0S_EINVAL, "bad precision %d", precision);
    if (bounds[0] != 0 || bounds[ntasks] != s) return fail(L0S_EINVAL, "bounds must run from 0 to s");
    for (int t = 0; t < ntasks; ++t)
        if (bounds[t + 1] < bounds[t]) return fail(L0S_EINVAL, "bounds must be non-decreasing");
    CK(cudaSetDevice(c->dev));
    c->staged = false;
    c->fix_on = false;
    c->m = m;
    c->s = s;
    c->T = ntasks;
    c->prec = precision;
    c->mp = ((m + 1 + 32 + 63) / 64) * 64;
    c->bounds_h.assign(bounds, bounds + ntasks + 1);
    c->zoff_h.assign((size_t)ntasks + 1, 0);
    c->rpad_h.assign((size_t)ntasks, 0);
    c->rows_h.assign((size_t)ntasks, 0.0);
    c->eta_h.assign((size_t)ntasks, 0.0);
    c->ld = 0;
    for (int t = 0; t < ntasks; ++t) {
        int64_t r = bounds[t + 1] - bounds[t];
        c->rpad_h[t] = ((r + 7) / 8) * 8;
        c->zoff_h[t + 1] = c->zoff_h[t] + c->rpad_h[t];
        c->rows_h[t] = (double)r;
        // per-entry bound on the normalized Gram error (error model):
        // dot products of length r over unit vectors (gamma_r) plus normalization
        c->eta_h[t] = 4.0 * (double)(r + 8) * kEps;
        c->ld = std::max(c->ld, r);
    }
    c->sp = std::max<int64_t>(c->zoff_h[ntasks], 8);
    size_t wsz = precision == L0S_PREC_FP32 ? 4 : 8;
    cudaEventRecord(c->ev[0], c->st);
    CK(c->bounds_d.ensure(sizeof(int64_t) * (ntasks + 1)));
    CK(c->zoff_d.ensure(sizeof(int64_t) * (ntasks + 1)));
    CK(cudaMemcpyAsync(c->bounds_d.p, bounds, sizeof(int64_t) * (ntasks + 1), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->zoff_d.p, c->zoff_h.data(), sizeof(int64_t) * (ntasks + 1), cudaMemcpyHostToDevice, c->st));
    CK(c->Xp.ensure(wsz * m * s));
    CK(c->yp.ensure(wsz * s));
    CK(c->Z.ensure(sizeof(double) * c->mp * c->sp));
    CK(c->G.ensure(sizeof(double) * c->mp * c->mp * ntasks));
    CK(c->qf.ensure(sizeof(double) * m * ntasks));
    CK(c->un2.ensure(sizeof(double) * m * ntasks));
    CK(c->yyu.ensure(sizeof(double) * ntasks));
    CK(c->rowsd.ensure(sizeof(double) * ntasks));
    CK(c->eta_d.ensure(sizeof(double) * ntasks));
    CK(cudaMemcpyAsync(c->rowsd.p, c->rows_h.data(), sizeof(double) * ntasks, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->eta_d.p, c->eta_h.data(), sizeof(double) * ntasks, cudaMemcpyHostToDevice, c->st));
    // rows past the property (m+1 .. mp-1) are Gram padding: zero; every other row of Z is
    // written whole (task padding included) by the normalize kernel
    CK(cudaMemsetAsync(c->Z.as<double>() + (m + 1) * c->sp, 0, sizeof(double) * (c->mp - m - 1) * c->sp, c->st));
    return L0S_OK;
}

static int gram_full(l0s_ctx* c);
static bool ozaki_planned(const l0s_ctx* c);

static OzFix oz_fix_of(l0s_ctx* c) {
    int* base = c->oz_fix.as<int>();
    return OzFix{base, base + l0s_ctx::kFixCap, l0s_ctx::kFixCap,
                 reinterpret_cast<unsigned char*>(base + l0s_ctx::kFixCap + 1)};
}

// the INT8 Gram's error bound with the loose rows left out when their (mean, scale) were stored
// (the staging kernels wrote the digits): k_oz_fixup then recomputes them in stage_post
static int ozaki_fix_prepare(l0s_ctx* c, OzFix* fx) {
    c->fix_on = c->digits_ready && c->oz_musc.p != nullptr;
    if (c->fix_on) {
        CK(c->oz_fix.ensure(sizeof(int) * (l0s_ctx::kFixCap + 1) + (size_t)(c->m + 1)));
        *fx = oz_fix_of(c);
    }
    return L0S_OK;
}

static int ozaki_eta(l0s_ctx* c, int T, int64_t m, int64_t mp) {
    OzFix fx{};
    const int rc = ozaki_fix_prepare(c, &fx);
    if (rc) return rc;
    launch_ozaki_eta(T, m, mp, c->oz_ex.as<int>(), c->rowsd.as<double>(), c->G.as<double>(), c->eta_d.as<double>(),
                     c->st, c->fix_on ? &fx : nullptr);
    return L0S_OK;
}

// stage after the Gram: unit diagonal, per-feature conditioning flags, host copies
static int stage_post(l0s_ctx* c) {
    const int64_t m = c->m;
    const int ntasks = c->T;
    cudaEventRecord(c->sev[3], c->st);
    if (c->gram_ozaki && c->fix_on)  // loose rows of the INT8 Gram: their fp64 rows first
        launch_ozaki_fixup(c->Xp.p, c->yp.p, c->prec, m, c->s, c->bounds_d.as<int64_t>(), ntasks,
                           c->oz_musc.as<double>(), (c->mp + 127) / 128 * 128, c->mp, oz_fix_of(c), c->G.as<double>(),
                           c->st);
    launch_unit_diag(c->G.as<double>(), ntasks, m, c->mp, c->st);
    CK(cudaGetLastError());
    // per-feature conditioning flags on the device (stage.cu: launch_feature_flags)
    CK(c->rho.ensure(sizeof(double) * m * ntasks));
    CK(c->rho_cap.ensure(sizeof(double) * ntasks));
    CK(c->ynorm.ensure(sizeof(double) * ntasks));
    CK(c->umin.ensure(sizeof(double) * ntasks));
    CK(c->iforce.ensure((size_t)m));
    CK(c->dead.ensure((size_t)m));
    launch_feature_flags(c->prec == L0S_PREC_FP32 ? 1e-5 : 1e-10, c->prec == L0S_PREC_FP32, c->qf.as<double>(), c->un2.as<double>(), c->rowsd.as<double>(), m, c->mp, ntasks,
                         c->umin.as<double>(), c->rho.as<double>(), c->rho_cap.as<double>(),
                         c->dead.as<unsigned char>(), c->iforce.as<unsigned char>(), c->G.as<double>(),
                         c->yyu.as<double>(), c->ynorm.as<double>(), c->st);
    CK(cudaGetLastError());
    cudaEventRecord(c->ev[1], c->st);
    cudaEventRecord(c->sev[4], c->st);
    c->yyu_h.assign((size_t)ntasks, 0.0);
    CK(cudaMemcpyAsync(c->yyu_h.data(), c->yyu.p, sizeof(double) * ntasks, cudaMemcpyDeviceToHost, c->st));
    if (c->gram_ozaki)
        CK(cudaMemcpyAsync(c->eta_h.data(), c->eta_d.p, sizeof(double) * ntasks, cudaMemcpyDeviceToHost, c->st));
    c->fix_count = 0;
    if (c->gram_ozaki && c->fix_on)
        CK(cudaMemcpyAsync(&c->fix_count, c->oz_fix.as<int>() + l0s_ctx::kFixCap, sizeof(int), cudaMemcpyDeviceToHost,
                           c->st));
    CK(cudaStreamSynchronize(c->st));
    if (c->gram_ozaki) {
        // the INT8 Gram's error bound must stay well inside the screen's first-order regime;
        // spiky rows (max |z| close to 1) make it too loose: up to kFixCap such rows were
        // recomputed in fp64 above (k_oz_fixup), more redo the whole Gram in fp64 (DMMA)
        bool loose = c->fix_count > l0s_ctx::kFixCap;
        for (int t = 0; t < ntasks; ++t) loose |= !(c->eta_h[(size_t)t] <= OZ_ETA_MAX);
        if (loose) {
            for (int t = 0; t < ntasks; ++t) c->eta_h[(size_t)t] = 4.0 * (c->rows_h[(size_t)t] + 8.0) * kEps;
            CK(cudaMemcpyAsync(c->eta_d.p, c->eta_h.data(), sizeof(double) * ntasks, cudaMemcpyHostToDevice, c->st));
            const int prev = c->gram_mode;
            c->gram_mode = L0S_GRAM_DMMA;
            if (c->digits_ready)  // the INT8 path skipped Z: write it now for the DMMA Gram
                launch_normalize(c->Xp.p, c->yp.p, c->prec, m, c->s, c->bounds_d.as<int64_t>(), c->zoff_d.as<int64_t>(),
                                 ntasks, c->sp, c->Z.as<double>(), c->qf.as<double>(), c->un2.as<double>(),
                                 c->yyu.as<double>(), 0, m + 1, DigitOut{nullptr, 0, 0, nullptr, nullptr}, c->st);
            gram_full(c);
            c->gram_mode = prev;
            launch_unit_diag(c->G.as<double>(), ntasks, m, c->mp, c->st);
            launch_feature_flags(c->prec == L0S_PREC_FP32 ? 1e-5 : 1e-10, c->prec == L0S_PREC_FP32, c->qf.as<double>(), c->un2.as<double>(), c->rowsd.as<double>(), m, c->mp, ntasks,
                                 c->umin.as<double>(), c->rho.as<double>(), c->rho_cap.as<double>(),
                                 c->dead.as<unsigned char>(), c->iforce.as<unsigned char>(), c->G.as<double>(),
                                 c->yyu.as<double>(), c->ynorm.as<double>(), c->st);
            CK(cudaStreamSynchronize(c->st));
        }
    }
    c->ddg_ready = false;
    c->ms_gram = elapsed(c->ev[0], c->ev[1]);
    c->ms_gram_k = c->gram_timed ? elapsed(c->ev[2], c->ev[3]) : 0.0;
    c->gram_timed = false;
    c->staged = true;
    c->binom_m = -1;
    return L0S_OK;
}

// The whole Gram in one go: the INT8 Ozaki path (tcgen05) when selected, else DMMA.
static bool ozaki_planned(const l0s_ctx* c) {
    return c->gram_mode == L0S_GRAM_OZAKI || (c->gram_mode == L0S_GRAM_AUTO && c->m >= 256);
}

static int gram_full(l0s_ctx* c) {
    const int nb = (int)(c->mp / 64);
    c->gram_ozaki = false;
    c->fix_on = false;
    if (ozaki_planned(c)) {
        OzFix fx{};
        const int frc = ozaki_fix_prepare(c, &fx);
        if (frc) return frc;
        int64_t KP = 0;
        const int64_t qb = ozaki_q_bytes(c->mp, c->T, c->rpad_h.data(), &KP);
        const int64_t R = (c->mp + 127) / 128 * 128;
        CK(c->oz_q.ensure((size_t)qb));
        CK(c->oz_ex.ensure(sizeof(int) * c->T * R));
        CK(c->oz_koff.ensure(sizeof(int64_t) * (c->T + 1)));
        cudaEventRecord(c->ev[2], c->st);
        if (launch_ozaki_gram(c->Z.as<double>(), c->sp, c->zoff_d.as<int64_t>(), c->rpad_h.data(), c->T, c->m, c->mp,
                              c->rowsd.as<double>(), c->G.as<double>(), c->eta_d.as<double>(), c->oz_q.as<int8_t>(),
                              c->oz_ex.as<int>(), c->oz_koff.as<int64_t>(), c->digits_ready, c->st,
                              c->fix_on ? &fx : nullptr) == 0) {
            cudaEventRecord(c->ev[3], c->st);
            c->gram_timed = true;
            c->gram_ozaki = true;
            return L0S_OK;
        }
        c->fix_on = false;
    }
    cudaEventRecord(c->ev[2], c->st);
    launch_gram_cols(c->Z.as<double>(), c->sp, c->zoff_d.as<int64_t>(), c->T, c->mp, c->G.as<double>(), 0, nb, c->st);
    cudaEventRecord(c->ev[3], c->st);
    c->gram_timed = true;
    return L0S_OK;
}

// Inputs -> Z (the reference's _prepare plus centering / normalization), and -- with
// gram_cols -- the Gram, overlapped with the transfer: host inputs travel in kChunks row
// chunks (multiples of the Gram's 64-row blocks) on the copy stream while the compute stream
// gathers and normalizes each chunk as it lands and computes every Gram block whose later
// block-row it completes.  Only the last chunk's blocks remain after the copy.
// Host rows [r0, r1) of the input into in_values on stream `st`: one contiguous copy, or one
// copy per row when the caller passed row pointers (a SelectedSubspace's entries, never stacked).
static cudaError_t copy_rows(l0s_ctx* c, const double* values, const double* const* rows, int64_t r0, int64_t r1,
                             int64_t dst_row, cudaStream_t st) {
    const int64_t s = c->s;
    double* dst = c->in_values.as<double>() + dst_row * s;
    // pageable sources (plain numpy arrays, the pipeline's real input) stream through the pinned
    // ring with parallel host copies (hostcopy.cu); pinned ones go straight to the copy engine
    const double* probe = rows ? rows[r0] : values + r0 * s;
    if (r1 > r0 && (size_t)(r1 - r0) * s * sizeof(double) >= ((size_t)1 << 20) && !host_is_pinned(probe)) {
        if (!c->stager) c->stager = host_stager_create();
        if (c->stager) {
            auto row = [&](int64_t r) -> const void* { return rows ? rows[r0 + r] : values + (r0 + r) * s; };
            return host_stager_copy_rows(c->stager, dst, row, r1 - r0, sizeof(double) * s, st);
        }
    }
    if (!rows) return cudaMemcpyAsync(dst, values + r0 * s, sizeof(double) * (r1 - r0) * s, cudaMemcpyHostToDevice, st);
    for (int64_t r = r0; r < r1;) {
        int64_t e = r + 1;  // rows adjacent in host memory travel as one copy
        while (e < r1 && rows[e] == rows[e - 1] + s) ++e;
        const cudaError_t err =
            cudaMemcpyAsync(dst + (r - r0) * s, rows[r], sizeof(double) * (e - r) * s, cudaMemcpyHostToDevice, st);
        if (err != cudaSuccess) return err;
        r = e;
    }
    return cudaSuccess;
}

static int stage_fill(l0s_ctx* c, const double* values, const double* y, const int64_t* perm, int is_device,
                      bool gram_cols, const double* const* rows = nullptr) {
    const int64_t m = c->m, s = c->s;
    const int ntasks = c->T, precision = c->prec;
    const double *vd = values, *yd = y;
    const int64_t* pd = perm;
    c->host_staged = !is_device;
    if (!is_device) {
        CK(c->in_values.ensure(sizeof(double) * m * s));
        CK(c->in_y.ensure(sizeof(double) * s));
        CK(c->in_perm.ensure(sizeof(int64_t) * s));
        CK(cudaMemcpyAsync(c->in_y.p, y, sizeof(double) * s, cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(c->in_perm.p, perm, sizeof(int64_t) * s, cudaMemcpyHostToDevice, c->st));
        vd = c->in_values.as<double>();
        yd = c->in_y.as<double>();
        pd = c->in_perm.as<int64_t>();
    }
    c->src_values = vd;  // the inputs in the caller's sample order (l0s_residuals reads them)
    c->src_y = yd;
    c->src_perm = pd;
    // the INT8 Gram's digits come out of the normalize kernel (no second pass over Z)
    DigitOut dig{nullptr, 0, 0, nullptr, nullptr};
    c->digits_ready = false;
    if (gram_cols && ozaki_planned(c)) {
        int64_t KP = 0;
        const int64_t qb = ozaki_q_bytes(c->mp, ntasks, c->rpad_h.data(), &KP);
        const int64_t R = (c->mp + 127) / 128 * 128;
        CK(c->oz_q.ensure((size_t)qb));
        CK(c->oz_ex.ensure(sizeof(int) * ntasks * R));
        CK(c->oz_koff.ensure(sizeof(int64_t) * (ntasks + 1)));
        CK(c->oz_musc.ensure(sizeof(double) * 2 * ntasks * R));
        ozaki_prepare_digits(m, c->mp, ntasks, c->rpad_h.data(), c->oz_q.as<int8_t>(), c->oz_ex.as<int>(),
                             c->oz_koff.as<int64_t>(), &dig, c->st, c->oz_musc.as<double>());
        dig.write_z = false;  // the INT8 Gram reads the digits; Z is written only for a DMMA fallback
        c->digits_ready = true;
    }
    int64_t max_rows = 0;
    for (int t = 0; t < ntasks; ++t) max_rows = std::max<int64_t>(max_rows, c->bounds_h[(size_t)t + 1] - c->bounds_h[(size_t)t]);
    auto rows_to_z = [&](int64_t f0, int64_t f1) {
        launch_stage_rows(vd, yd, pd, m, s, precision, c->Xp.p, c->yp.p, c->bounds_d.as<int64_t>(),
                          c->zoff_d.as<int64_t>(), ntasks, c->sp, c->Z.as<double>(), c->qf.as<double>(),
                          c->un2.as<double>(), c->yyu.as<double>(), f0, f1, dig, max_rows, c->st);
    };
    const int nb = (int)(c->mp / 64);
    const bool chunked = !is_device && (double)m * (double)s * 8.0 >= 32.0 * (1 << 20) && m >= 2 * 64;
    rows_to_z(m, m + 1);  // the property first: every Gram column block needs it
    if (!chunked) {
        if (!is_device)
            CK(copy_rows(c, values, rows, 0, m, 0, c->st));
        // the staging pass timed (bench.py reports its HBM rate): sev[0..1] bracket it
        cudaEventRecord(c->sev[0], c->st);
        rows_to_z(0, m);
        cudaEventRecord(c->sev[1], c->st);
        cudaEventRecord(c->sev[2], c->st);
        c->stage_fused = stage_rows_fused(max_rows, dig);
        c->stage_timed = true;
        if (gram_cols) return gram_full(c);
        return L0S_OK;
    }
    c->stage_timed = false;
    // the INT8 Gram runs once all rows have landed
    const bool ozaki = gram_cols && c->digits_ready;
    if (ozaki) gram_cols = false;
    const int64_t R = (((m + l0s_ctx::kChunks - 1) / l0s_ctx::kChunks) + 63) / 64 * 64;
    // the copy stream starts after everything queued so far (buffers may be in use by a search)
    cudaEventRecord(c->cev[l0s_ctx::kChunks], c->st);
    cudaStreamWaitEvent(c->cst, c->cev[l0s_ctx::kChunks], 0);
    int k = 0;
    int oz_done = 0;  // INT8 Gram: column blocks (64 wide) already launched
    if (ozaki) {
        cudaEventRecord(c->ev[2], c->st);
        c->gram_timed = true;
        c->gram_ozaki = true;
    }
    // chunk k's copy is issued, then its compute is queued behind it: from pageable memory the
    // host is busy copying chunk k + 1 into the pinned ring while the device stages chunk k
    for (int64_t r0 = 0; r0 < m; r0 += R, ++k) {
        const int64_t r1 = std::min(m, r0 + R);
        CK(copy_rows(c, values, rows, r0, r1, r0, c->cst));
        cudaEventRecord(c->cev[k], c->cst);
        cudaStreamWaitEvent(c->st, c->cev[k], 0);
        rows_to_z(r0, r1);
        if (gram_cols) {
            const int B0 = (int)(r0 / 64), B1 = r1 >= m ? nb : (int)(r1 / 64);
            launch_gram_cols(c->Z.as<double>(), c->sp, c->zoff_d.as<int64_t>(), ntasks, c->mp, c->G.as<double>(),
                             B0, B1, c->st);
        }
        if (ozaki) {
            // a column block is complete once every row its tiles cover has landed (ozaki_blocks_ready)
            const int ncb = ozaki_col_blocks(c->mp);
            const int upto = r1 >= m ? ncb : std::max(oz_done, std::min(ncb, ozaki_blocks_ready(r1)));
            if (launch_ozaki_tiles(ntasks, c->mp, c->rpad_h.data(), c->oz_q.as<int8_t>(), c->oz_ex.as<int>(),
                                   c->oz_koff.as<int64_t>(), c->G.as<double>(), oz_done, upto, c->st))
                return fail(L0S_ECUDA, "INT8 Gram: TMA descriptor");
            oz_done = upto;
        }
    }
    if (ozaki) {
        const int rc = ozaki_eta(c, ntasks, m, c->mp);
        if (rc) return rc;
        cudaEventRecord(c->ev[3], c->st);
    }
    return L0S_OK;
}

int l0s_stage(l0s_ctx* c, const double* values, int64_t m, int64_t s, const double* y, const int64_t* perm,
              const int64_t* bounds, int ntasks, int precision, int is_device) {
    int rc = stage_prepare(c, values, m, s, y, perm, bounds, ntasks, precision, is_device);
    if (rc) return rc;
    rc = stage_fill(c, values, y, perm, is_device, true);
    if (rc) return rc;
    CK(cudaGetLastError());
    return stage_post(c);
}

int l0s_stage_rows(l0s_ctx* c, const double* const* rows, int64_t m, int64_t s, const double* y, const int64_t* perm,
                   const int64_t* bounds, int ntasks, int precision) {
    if (!rows && m > 0) return fail(L0S_EINVAL, "null row pointers");
    for (int64_t r = 0; r < m; ++r)
        if (!rows[r]) return fail(L0S_EINVAL, "row %lld: null pointer", (long long)r);
    int rc = stage_prepare(c, nullptr, m, s, y, perm, bounds, ntasks, precision, 0);
    if (rc) return rc;
    rc = stage_fill(c, nullptr, y, perm, 0, true, rows);
    if (rc) return rc;
    CK(cudaGetLastError());
    return stage_post(c);
}

// Incremental stage across the pipeline's dimensions: the subspace only grows
// by appending (screening.py:197-198), so only the new rows cross PCIe; the device keeps the
// previous inputs and restages from them (gather, normalize, Gram and flags are device work:
// 0.6 ms at C3 against 2.9 ms for the copy of the old rows).
static int stage_append(l0s_ctx* c, const double* values, const double* const* rows, int64_t m_new);

int l0s_stage_append(l0s_ctx* c, const double* rows, int64_t m_new) { return stage_append(c, rows, nullptr, m_new); }

int l0s_stage_append_rows(l0s_ctx* c, const double* const* rows, int64_t m_new) {
    if (!rows && m_new > 0) return fail(L0S_EINVAL, "null row pointers");
    for (int64_t r = 0; r < m_new; ++r)
        if (!rows[r]) return fail(L0S_EINVAL, "row %lld: null pointer", (long long)r);
    return stage_append(c, nullptr, rows, m_new);
}

// Extend a staged problem (INT8 Gram) from m0 to m1 features whose new rows already sit in
// in_values: the old feature block of the Gram, the old rows of Z / Xp, their INT8 digits and
// exponents and their per-task norms move to the new layout (device copies, the property row
// is re-staged at index m1), only the new rows are gathered and normalized, and only the Gram
// column blocks that hold a new column (and the property's) are recomputed -- every entry of the
// INT8 Gram depends only on its two rows' digits, so the result is the full stage's bit for bit.
static int stage_extend(l0s_ctx* c, int64_t m1) {
    const int64_t m0 = c->m, s = c->s, sp = c->sp;
    const int T = c->T;
    const int64_t mp0 = c->mp, mp1 = ((m1 + 1 + 32 + 63) / 64) * 64;
    const int64_t R0 = (mp0 + 127) / 128 * 128, R1 = (mp1 + 127) / 128 * 128;
    const size_t wsz = c->prec == L0S_PREC_FP32 ? 4 : 8;
    int64_t KP = 0;
    const int64_t qb1 = ozaki_q_bytes(mp1, T, c->rpad_h.data(), &KP);
    cudaEventRecord(c->ev[0], c->st);
    // relayout into fresh buffers (old contents copied), then swap
    DBuf G1, Q1, ex1, qf1, un21, ms1;
    CK(G1.ensure(sizeof(double) * mp1 * mp1 * T));
    CK(Q1.ensure((size_t)qb1));
    CK(ex1.ensure(sizeof(int) * T * R1));
    const bool musc = c->oz_musc.p != nullptr;
    if (musc) CK(ms1.ensure(sizeof(double) * 2 * T * R1));
    CK(qf1.ensure(sizeof(double) * m1 * T));
    CK(un21.ensure(sizeof(double) * m1 * T));
    for (int t = 0; t < T; ++t) {
        CK(cudaMemcpy2DAsync(G1.as<double>() + (int64_t)t * mp1 * mp1, sizeof(double) * mp1,
                             c->G.as<double>() + (int64_t)t * mp0 * mp0, sizeof(double) * mp0, sizeof(double) * m0,
                             (size_t)m0, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(ex1.as<int>() + (int64_t)t * R1, c->oz_ex.as<int>() + (int64_t)t * R0, sizeof(int) * m0,
                           cudaMemcpyDeviceToDevice, c->st));
        if (musc)
            CK(cudaMemcpyAsync(ms1.as<double>() + 2 * (int64_t)t * R1, c->oz_musc.as<double>() + 2 * (int64_t)t * R0,
                               sizeof(double) * 2 * m0, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(qf1.as<double>() + (int64_t)t * m1, c->qf.as<double>() + (int64_t)t * m0,
                           sizeof(double) * m0, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(un21.as<double>() + (int64_t)t * m1, c->un2.as<double>() + (int64_t)t * m0,
                           sizeof(double) * m0, cudaMemcpyDeviceToDevice, c->st));
    }
    for (int a = 0; a < OZ_DIGITS; ++a)
        CK(cudaMemcpyAsync(Q1.as<int8_t>() + (int64_t)a * R1 * KP, c->oz_q.as<int8_t>() + (int64_t)a * R0 * KP,
                           (size_t)(m0 * KP), cudaMemcpyDeviceToDevice, c->st));
    std::swap(c->G, G1);
    std::swap(c->oz_q, Q1);
    std::swap(c->oz_ex, ex1);
    if (musc) std::swap(c->oz_musc, ms1);
    std::swap(c->qf, qf1);
    std::swap(c->un2, un21);
    CK(cudaStreamSynchronize(c->st));  // the old buffers are released on return
    CK(c->Z.grow(sizeof(double) * mp1 * sp, sizeof(double) * m0 * sp, c->st));
    CK(c->Xp.grow(wsz * m1 * s, wsz * m0 * s, c->st));
    c->m = m1;
    c->mp = mp1;
    c->staged = false;
    CK(cudaMemsetAsync(c->Z.as<double>() + (m1 + 1) * sp, 0, sizeof(double) * (mp1 - m1 - 1) * sp, c->st));
    // digit rows past the property (padding) and their exponents: zero
    for (int a = 0; a < OZ_DIGITS; ++a)
        CK(cudaMemsetAsync(c->oz_q.as<int8_t>() + ((int64_t)a * R1 + m1 + 1) * KP, 0, (size_t)((R1 - m1 - 1) * KP), c->st));
    for (int t = 0; t < T; ++t)
        CK(cudaMemsetAsync(c->oz_ex.as<int>() + (int64_t)t * R1 + m1 + 1, 0, sizeof(int) * (R1 - m1 - 1), c->st));
    DigitOut dig{c->oz_q.as<int8_t>(), R1, KP, c->oz_koff.as<int64_t>(), c->oz_ex.as<int>(), false,
                 musc ? c->oz_musc.as<double>() : nullptr};
    const double* vd = c->in_values.as<double>();
    const double* yd = c->in_y.as<double>();
    const int64_t* pd = c->in_perm.as<int64_t>();
    for (int64_t f0 : {m1, m0}) {  // the property (row m1), then the new features (rows m0 .. m1-1)
        const int64_t f1 = f0 == m1 ? m1 + 1 : m1;
        int64_t max_rows = 0;
        for (int t = 0; t < T; ++t) max_rows = std::max<int64_t>(max_rows, c->bounds_h[(size_t)t + 1] - c->bounds_h[(size_t)t]);
        launch_stage_rows(vd, yd, pd, m1, s, c->prec, c->Xp.p, c->yp.p, c->bounds_d.as<int64_t>(),
                          c->zoff_d.as<int64_t>(), T, sp, c->Z.as<double>(), c->qf.as<double>(), c->un2.as<double>(),
                          c->yyu.as<double>(), f0, f1, dig, max_rows, c->st);
    }
    // column blocks holding a new column or the property's (their tiles cover every row)
    cudaEventRecord(c->ev[2], c->st);
    if (launch_ozaki_tiles(T, mp1, c->rpad_h.data(), c->oz_q.as<int8_t>(), c->oz_ex.as<int>(),
                           c->oz_koff.as<int64_t>(), c->G.as<double>(), (int)(m0 / 128), ozaki_col_blocks(mp1), c->st))
        return fail(L0S_ECUDA, "INT8 Gram: TMA descriptor");
    // the per-task entry bound over every row's exponent (old rows' exponents moved above)
    {
        const int rc = ozaki_eta(c, T, m1, mp1);
        if (rc) return rc;
    }
    cudaEventRecord(c->ev[3], c->st);
    c->gram_timed = true;
    c->gram_ozaki = true;
    c->stage_timed = false;
    c->binom_m = -1;
    CK(cudaGetLastError());
    const int rc = stage_post(c);
    c->host_staged = true;
    return rc;
}

static int stage_append(l0s_ctx* c, const double* values, const double* const* rows, int64_t m_new) {
    if (!c) return fail(L0S_EINVAL, "null context");
    if (!c->staged || !c->host_staged || c->shard_pending)
        return fail(L0S_ESTATE, "l0s_stage_append needs a completed stage from host inputs");
    if (m_new < 0) return fail(L0S_EINVAL, "m_new must be >= 0");
    if (m_new == 0) return L0S_OK;
    CK(cudaSetDevice(c->dev));
    const int64_t m0 = c->m, s = c->s, m1 = m0 + m_new;
    CK(cudaStreamSynchronize(c->st));
    CK(c->in_values.grow(sizeof(double) * m1 * s, sizeof(double) * m0 * s, c->st));
    CK(copy_rows(c, values, rows, 0, m_new, m0, c->st));
    if (c->gram_ozaki && c->digits_ready && c->gram_mode != L0S_GRAM_DMMA) return stage_extend(c, m1);
    const std::vector<int64_t> bounds = c->bounds_h;
    int rc = stage_prepare(c, c->in_values.as<double>(), m1, s, c->in_y.as<double>(), c->in_perm.as<int64_t>(),
                           bounds.data(), c->T, c->prec, 1);
    if (rc) return rc;
    rc = stage_fill(c, c->in_values.as<double>(), c->in_y.as<double>(), c->in_perm.as<int64_t>(), 1, true);
    if (rc) return rc;
    CK(cudaGetLastError());
    rc = stage_post(c);
    c->host_staged = true;  // the inputs are still ours
    return rc;
}

int l0s_gram_shard_size(int64_t m, int ntasks, int nshards, int64_t* out_doubles) {
    if (m < 1 || ntasks < 1 || nshards < 1) return fail(L0S_EINVAL, "need m, ntasks, nshards >= 1");
    const int64_t mp = ((m + 1 + 32 + 63) / 64) * 64;
    *out_doubles = gram_shard_blocks(mp, ntasks, nshards) * 64 * 64;
    return L0S_OK;
}

int l0s_stage_shard(l0s_ctx* c, const double* values, int64_t m, int64_t s, const double* y, const int64_t* perm,
                    const int64_t* bounds, int ntasks, int precision, int is_device, int shard, int nshards,
                    double* pack) {
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(L0S_EINVAL, "shard %d of %d", shard, nshards);
    if (nshards > 1 && !pack) return fail(L0S_EINVAL, "pack buffer required for nshards > 1");
    int rc = stage_prepare(c, values, m, s, y, perm, bounds, ntasks, precision, is_device);
    if (rc) return rc;
    rc = stage_fill(c, values, y, perm, is_device, nshards == 1);
    if (rc) return rc;
    if (nshards > 1)
        launch_gram(c->Z.as<double>(), c->sp, c->zoff_d.as<int64_t>(), ntasks, c->mp, c->G.as<double>(), shard,
                    nshards, pack, c->st);
    CK(cudaGetLastError());
    if (nshards == 1) return stage_post(c);
    CK(cudaStreamSynchronize(c->st));  // the pack is complete for the caller's all-gather
    c->shard_pending = true;
    return L0S_OK;
}

int l0s_stage_finish(l0s_ctx* c, const double* gathered) {
    if (!c || !c->shard_pending) return fail(L0S_ESTATE, "l0s_stage_shard (nshards > 1) must come first");
    if (!gathered) return fail(L0S_EINVAL, "null gathered buffer");
    CK(cudaSetDevice(c->dev));
    launch_gram_unpack(gathered, c->T, c->mp, c->G.as<double>(), c->st);
    CK(cudaGetLastError());
    c->shard_pending = false;
    return stage_post(c);
}

int l0s_count(int64_t m, int n, int64_t* out) {
    if (n < 1 || m < 0) return fail(L0S_EINVAL, "need m >= 0 and n >= 1");
    int64_t v = binom_sat(m, n);
    if (v == INT64_MAX) return fail(L0S_ECAPACITY, "C(%lld, %d) exceeds the enumerable range", (long long)m, n);
    *out = v;
    return L0S_OK;
}

int l0s_unrank(int64_t rank, int64_t m, int n, int64_t* out) {
    int64_t total;
    int rc = l0s_count(m, n, &total);
    if (rc) return rc;
    if (rank < 0 || rank >= total) return fail(L0S_EINVAL, "rank %lld outside [0, %lld)", (long long)rank, (long long)total);
    int64_t r = rank, e = 0;
    for (int k = 0; k < n; ++k) {
        int rem = n - k - 1;
        for (;;) {
            int64_t cc = binom_sat(m - 1 - e, rem);
            if (r < cc) break;
            r -= cc;
            ++e;
        }
        out[k] = e++;
    }
    return L0S_OK;
}

int l0s_rank(const int64_t* tup, int64_t m, int n, int64_t* out) {
    int64_t total;
    int rc = l0s_count(m, n, &total);
    if (rc) return rc;
    int64_t prev = -1;
    for (int k = 0; k < n; ++k) {
        if (!(prev < tup[k] && tup[k] < m)) return fail(L0S_EINVAL, "tuple is not strictly increasing within range");
        prev = tup[k];
    }
    // rank = C(m,n) - 1 - sum_k C(m-1-c_k, n-k)
    int64_t acc = 0;
    for (int k = 0; k < n; ++k) acc += binom_sat(m - 1 - tup[k], n - k);
    *out = total - 1 - acc;
    return L0S_OK;
}

int l0s_fit_tuples(l0s_ctx* c, int n, const int64_t* tuples, int64_t count, int32_t* out_ok, double* out_score,
                   double* out_coef, double* out_ssr) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (n < 1 || n > 15) return fail(L0S_EINVAL, "dimension %d outside [1, 15]", n);
    if (count <= 0) return L0S_OK;
    CK(cudaSetDevice(c->dev));
    for (int64_t i = 0; i < count; ++i)
        for (int k = 0; k < n; ++k) {
            int64_t v = tuples[i * n + k];
            if (v < 0 || v >= c->m || (k > 0 && v <= tuples[i * n + k - 1]))
                return fail(L0S_EINVAL, "tuple %lld is not strictly increasing within [0, %lld)", (long long)i, (long long)c->m);
        }
    int rc = ensure_binom(c, n);
    if (rc) return rc;
    CK(c->ex_tuples.ensure(sizeof(int64_t) * count * n));
    CK(cudaMemcpyAsync(c->ex_tuples.p, tuples, sizeof(int64_t) * count * n, cudaMemcpyHostToDevice, c->st));
    rc = run_exact(c, n, nullptr, c->ex_tuples.as<int64_t>(), count, true, nullptr);
    if (rc) return rc;
    const int p = n + 1;
    if (out_ok) CK(cudaMemcpyAsync(out_ok, c->ex_ok.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, c->st));
    if (out_score) CK(cudaMemcpyAsync(out_score, c->ex_score.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->st));
    if (out_coef) CK(cudaMemcpyAsync(out_coef, c->ex_coef.p, sizeof(double) * count * c->T * p, cudaMemcpyDeviceToHost, c->st));
    if (out_ssr) CK(cudaMemcpyAsync(out_ssr, c->ex_ssr.p, sizeof(double) * count * c->T, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

static void fill_fit_common(l0s_ctx* c, FitArgs& a, int n) {
    a.G = c->G.as<double>();
    a.qf = c->qf.as<double>();
    a.un2 = c->un2.as<double>();
    a.rowsd = c->rowsd.as<double>();
    a.eta = c->eta_d.as<double>();
    a.rho = c->rho.as<double>();
    a.rho_cap = c->rho_cap.as<double>();
    a.ynorm = c->ynorm.as<double>();
    a.iforce = c->iforce.as<unsigned char>();
    a.n = n;
    a.binom = c->binom.as<int64_t>();
    a.m = c->m;
    a.mp = c->mp;
    a.T = c->T;
    a.N_total = binom_sat(c->m, n);
    double tol = c->prec == L0S_PREC_FP32 ? 1e-5 : 1e-10;
    a.tol2 = tol * tol;
    a.ref_fp32 = c->prec == L0S_PREC_FP32 ? 1 : 0;
}

int l0s_screen_tuples(l0s_ctx* c, int n, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (n < 2 || n > 5) return fail(L0S_EINVAL, "screened bounds are implemented for n = 2 to 5");
    if (count <= 0) return L0S_OK;
    CK(cudaSetDevice(c->dev));
    int rc = ensure_binom(c, n);
    if (rc) return rc;
    FitArgs a{};
    fill_fit_common(c, a, n);
    CK(c->ex_tuples.ensure(sizeof(int64_t) * count * n));
    CK(c->cand_lb.ensure(sizeof(double) * count));
    CK(c->ex_ok.ensure(sizeof(int32_t) * count));
    CK(cudaMemcpyAsync(c->ex_tuples.p, tuples, sizeof(int64_t) * count * n, cudaMemcpyHostToDevice, c->st));
    if (n == 2)
        launch_screen2(a, c->ex_tuples.as<int64_t>(), count, c->cand_lb.as<double>(), c->ex_ok.as<int32_t>(), c->st);
    else if (n == 3)
        launch_screen3(a, c->ex_tuples.as<int64_t>(), count, c->cand_lb.as<double>(), c->ex_ok.as<int32_t>(), c->st);
    else if (n == 4)
        launch_screen4(a, c->ex_tuples.as<int64_t>(), count, c->cand_lb.as<double>(), c->ex_ok.as<int32_t>(), c->st);
    else
        launch_screen5(a, c->ex_tuples.as<int64_t>(), count, c->cand_lb.as<double>(), c->ex_ok.as<int32_t>(), c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_lb, c->cand_lb.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(out_flags, c->ex_ok.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

static int run_qr_screen(l0s_ctx* c, QrArgs& q, int n, int64_t count, int64_t* launches, bool allow_dd);

int l0s_qr_tuples(l0s_ctx* c, int n, const int64_t* tuples, int64_t count, double* out_score, double* out_ratio) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (n < 1 || n > 6) return fail(L0S_EINVAL, "the QR screen takes n in [1, 6]");
    if (count <= 0) return L0S_OK;
    CK(cudaSetDevice(c->dev));
    int rc = ensure_binom(c, n);
    if (rc) return rc;
    std::vector<int64_t> rk((size_t)count);
    for (int64_t i = 0; i < count; ++i) {
        rc = l0s_rank(tuples + i * n, c->m, n, &rk[(size_t)i]);
        if (rc) return rc;
    }
    CK(c->ex_ranks.ensure(sizeof(int64_t) * count));
    CK(c->qr_ssr.ensure(sizeof(double) * count * c->T));
    CK(c->qr_ratio.ensure(sizeof(double) * count * c->T));
    CK(c->qr_score.ensure(sizeof(double) * count));
    CK(c->qr_minr.ensure(sizeof(double) * count));
    CK(cudaMemcpyAsync(c->ex_ranks.p, rk.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice, c->st));
    QrArgs q{};
    q.Xp = c->Xp.as<double>();
    q.yp = c->yp.as<double>();
    q.bounds = c->bounds_d.as<int64_t>();
    q.T = c->T;
    q.m = c->m;
    q.s = c->s;
    q.n = n;
    q.ranks = c->ex_ranks.as<int64_t>();
    q.binom = c->binom.as<int64_t>();
    q.ssr = c->qr_ssr.as<double>();
    q.ratio = c->qr_ratio.as<double>();
    q.score = c->qr_score.as<double>();
    q.min_ratio = c->qr_minr.as<double>();
    rc = run_qr_screen(c, q, n, count, nullptr, false);  // diagnostics: TSQR unless L0S_QR_SCREEN=dd
    if (rc) return rc;
    CK(cudaMemcpyAsync(out_score, c->qr_score.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(out_ratio, c->qr_minr.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

int l0s_residuals(l0s_ctx* c, int n, const int64_t* tuples, const double* coef, int64_t count, double* out) {
    if (!c || !c->staged || !c->src_values) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (n < 1 || n > 15) return fail(L0S_EINVAL, "dimension %d outside [1, 15]", n);
    if (count <= 0) return L0S_OK;
    for (int64_t i = 0; i < count * n; ++i)
        if (tuples[i] < 0 || tuples[i] >= c->m) return fail(L0S_EINVAL, "feature index outside the staged subspace");
    CK(cudaSetDevice(c->dev));
    const int p = n + 1;
    CK(c->res_tup.ensure(sizeof(int64_t) * count * n));
    CK(c->res_coef.ensure(sizeof(double) * count * c->T * p));
    CK(c->res_out.ensure(sizeof(double) * count * c->s));
    CK(cudaMemcpyAsync(c->res_tup.p, tuples, sizeof(int64_t) * count * n, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->res_coef.p, coef, sizeof(double) * count * c->T * p, cudaMemcpyHostToDevice, c->st));
    launch_residuals(c->src_values, c->src_y, c->src_perm, c->bounds_d.as<int64_t>(), c->T, c->s, n,
                     c->res_tup.as<int64_t>(), c->res_coef.as<double>(), count, c->res_out.as<double>(), c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, c->res_out.p, sizeof(double) * count * c->s, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

int l0s_get_gram(l0s_ctx* c, int task, double* out) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (task < 0 || task >= c->T) return fail(L0S_EINVAL, "task out of range");
    CK(cudaSetDevice(c->dev));
    int64_t w = c->m + 1;
    CK(cudaMemcpy2DAsync(out, sizeof(double) * w, c->G.as<double>() + (int64_t)task * c->mp * c->mp,
                         sizeof(double) * c->mp, sizeof(double) * w, (size_t)w, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

// ---------------------------------------------------------------------------
// the search
// ---------------------------------------------------------------------------

static int search_exact_mode(l0s_ctx* c, int n, int64_t keep, int64_t rb, int64_t re, std::vector<Cand>& best,
                             l0s_stats* st) {
    // every tuple through the bit-exact kernel, chunked; per chunk the device sorts the scores
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(re - rb, (int64_t)1 << 20));
    CK(c->ex_ranks.ensure(sizeof(int64_t) * chunk));
    CK(c->lb_tmp.ensure(sizeof(double) * chunk));
    CK(c->rank_tmp.ensure(sizeof(int64_t) * chunk));
    size_t tb = sort_pairs_temp_bytes(chunk);
    CK(c->sort_tmp.ensure(tb));
    for (int64_t r0 = rb; r0 < re; r0 += chunk) {
        int64_t cnt = std::min(chunk, re - r0);
        k_iota<<<(unsigned)((cnt + 255) / 256), 256, 0, c->st>>>(c->ex_ranks.as<int64_t>(), r0, cnt);
        st->n_launches++;
        int rc = run_exact(c, n, c->ex_ranks.as<int64_t>(), nullptr, cnt, false, &st->n_launches);
        if (rc) return rc;
        // sort (score, rank) on device; non-finite scores sort last (ord_enc maps +inf above all finite)
        const int ns = sort_pairs(c->ex_score.as<double>(), c->ex_ranks.as<int64_t>(), c->lb_tmp.as<double>(),
                                  c->rank_tmp.as<int64_t>(), cnt, c->sort_tmp.p, tb, c->st);
        if (ns < 0) return fail(L0S_ECUDA, "sort scratch too small");
        st->n_launches += ns;
        // sorted by (score, rank): the first `keep` entries are the chunk's best in the
        // reference's order (search.py:303); non-finite scores sort last
        int64_t take = std::min<int64_t>(cnt, keep);
        std::vector<double> sc((size_t)take);
        std::vector<int64_t> rk((size_t)take);
        CK(cudaMemcpyAsync(sc.data(), c->ex_score.p, sizeof(double) * take, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(rk.data(), c->ex_ranks.p, sizeof(int64_t) * take, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        std::vector<Cand> more;
        for (int64_t i = 0; i < take; ++i) more.push_back({sc[(size_t)i], rk[(size_t)i]});
        merge_best(best, more, keep);
    }
    st->mode_used = L0S_MODE_EXACT;
    st->certified = 1;
    return L0S_OK;
}

// QR screen of the `nill` ranks in c->ill, then bit-exact refit of the ones that can matter.
// L0S_QR_SCREEN=dd | tsqr forces the ill-tuple screen (tests, experiments); else chosen by cost
static int qr_screen_forced() {
    const char* e = getenv("L0S_QR_SCREEN");
    return !e ? 0 : (!strcmp(e, "dd") ? 2 : (!strcmp(e, "tsqr") ? 1 : 0));
}

// the QR screen of `count` ranks already in q.ranks (scores and min ratios in q.score / q.min_ratio)
static int run_qr_screen(l0s_ctx* c, QrArgs& q, int n, int64_t count, int64_t* launches, bool allow_dd) {
    const int forced = qr_screen_forced();
    bool dd = forced == 2 || (forced == 0 && allow_dd && dd_screen_pays(count, n, c->T, c->m, c->s));
    if (dd) {
        const int64_t LD = dd_gram_ld(c->m);
        const size_t bytes = sizeof(double) * (size_t)c->T * LD * LD;
        dd = c->ddg_hi.ensure(bytes) == cudaSuccess &&
             c->ddg_lo.ensure(sizeof(double) * (size_t)dd_gram_lo_doubles(c->m, c->T)) == cudaSuccess;
        if (!dd) cudaGetLastError();
    }
    if (dd) {
        launch_dd_screen(q, count, c->ddg_hi.as<double>(), c->ddg_lo.as<double>(), c->ddg_ready, c->st, launches);
        c->ddg_ready = true;
        q.total = count * q.T;
        launch_qr_finalize(q, count, c->st, launches);
    } else {
        launch_qr_screen(q, count, c->st, launches);
    }
    CK(cudaGetLastError());
    return L0S_OK;
}

static int screen_ill(l0s_ctx* c, int n, int64_t nill, int64_t keep, std::vector<Cand>& best, l0s_stats* st,
                      double cap = INFINITY) {
    if (c->prec == L0S_PREC_FP32) {
        // the fp64 QR screen cannot bound the reference's float32 arithmetic on an
        // ill-conditioned system: every such tuple is refit bit-exactly
        st->n_ill_refit += nill;
        std::vector<Cand> more;
        int rc = exact_ranks_to_host(c, n, c->ill.as<int64_t>(), nill, more, &st->n_launches, &c->recs);
        if (rc) return rc;
        st->n_candidates += nill;
        merge_best(best, more, keep);
        return L0S_OK;
    }
    CK(c->qr_ssr.ensure(sizeof(double) * nill * c->T));
    CK(c->qr_ratio.ensure(sizeof(double) * nill * c->T));
    CK(c->qr_score.ensure(sizeof(double) * nill));
    CK(c->qr_minr.ensure(sizeof(double) * nill));
    QrArgs q{};
    q.Xp = c->Xp.as<double>();
    q.yp = c->yp.as<double>();
    q.bounds = c->bounds_d.as<int64_t>();
    q.T = c->T;
    q.m = c->m;
    q.s = c->s;
    q.n = n;
    q.ranks = c->ill.as<int64_t>();
    q.binom = c->binom.as<int64_t>();
    q.ssr = c->qr_ssr.as<double>();
    q.ratio = c->qr_ratio.as<double>();
    q.score = c->qr_score.as<double>();
    q.min_ratio = c->qr_minr.as<double>();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c->st);
    // many ill tuples: one double-double Gram of every column, then a (n + 2)-block LDL^T per
    // tuple (ddgram.cu); few: the TSQR screen reads each tuple's columns
    {
        const int rc = run_qr_screen(c, q, n, nill, &st->n_launches, true);
        if (rc) return rc;
    }
    cudaEventRecord(e1, c->st);
    CK(cudaGetLastError());
    CK(cudaEventSynchronize(e1));
    st->ms_qr += elapsed(e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double tol = 1e-10;  // RANK_TOL_FACTOR["fp64"], lsq.py:23 (fp32 never reaches the QR screen)
    double yy = 0.0;
    for (double v : c->yyu_h) yy += v;
    const double sk = std::min(((int64_t)best.size() >= keep) ? best[(size_t)keep - 1].score : INFINITY, cap);
    // selection on the device: only the (usually empty) list of survivors comes back
    CK(c->ex_ranks.ensure(sizeof(int64_t) * (size_t)std::max<int64_t>(nill, 1)));
    CK(c->cand_cnt.ensure(sizeof(unsigned long long)));
    CK(cudaMemsetAsync(c->cand_cnt.p, 0, sizeof(unsigned long long), c->st));
    launch_qr_select(q.score, q.min_ratio, c->ill.as<int64_t>(), nill, tol, sk, yy / (double)c->s,
                     c->ex_ranks.as<int64_t>(), c->cand_cnt.as<unsigned long long>(), nill, c->st);
    st->n_launches++;
    unsigned long long nsel = 0;
    CK(cudaMemcpyAsync(&nsel, c->cand_cnt.p, sizeof nsel, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    std::vector<int64_t> sel((size_t)nsel);
    if (nsel) CK(cudaMemcpy(sel.data(), c->ex_ranks.p, sizeof(int64_t) * nsel, cudaMemcpyDeviceToHost));
    st->n_ill_refit += (int64_t)sel.size();
    if (sel.empty()) return L0S_OK;
    std::vector<Cand> more;
    int rc = exact_ranks_to_host(c, n, c->ex_ranks.as<int64_t>(), (int64_t)sel.size(), more, &st->n_launches, &c->recs);
    if (rc) return rc;
    st->n_candidates += (int64_t)sel.size();
    merge_best(best, more, keep);
    return L0S_OK;
}

static int search_fast_mode(l0s_ctx* c, int n, int64_t keep, int64_t rb, int64_t re, std::vector<Cand>& best,
                            l0s_stats* st) {
    const int64_t N = binom_sat(c->m, n);
    // unit table (cached per problem shape, rank range and part)
    int64_t key[7] = {c->m, c->T, rb, re, n, c->part, c->nparts};
    if (!std::equal(key, key + 7, c->units_key)) {
        // prefix[v] = rank of the first tuple whose smallest index is v
        std::vector<int64_t> pre((size_t)c->m + 1, 0);
        for (int64_t v = 0; v < c->m; ++v) pre[(size_t)v + 1] = pre[(size_t)v] + binom_sat(c->m - 1 - v, n - 1);
        c->units_h = n == 2 ? fit2_units(c->m, pre, rb, re)
                     : n == 3 ? fit3_units(c->m, c->T, N, pre, rb, re, c->nparts == 1)
                     : n == 4 ? fit4_units(c->m, c->T, pre, rb, re)
                              : fit5_units(c->m, c->T, pre, rb, re);
        if (c->nparts > 1) {
            // a part gets 1/nparts of the units: split their i ranges until every part still has
            // several units per CTA, then deal them round-robin over the longest-first order
            // from shared values only (not this device's SM count or occupancy): every rank must
            // build the same split table, or parts would overlap or leave gaps
            const int g = kPartGridCtas;
            int64_t rows = 0;
            for (const int4& u : c->units_h) rows += u.w - u.z;
            const int64_t target = (int64_t)6 * g * c->nparts;
            const int ich = (int)std::max<int64_t>(64, (rows / std::max<int64_t>(target, 1) + 31) / 32 * 32);
            std::vector<int4> split;
            for (const int4& u : c->units_h)
                for (int lo = u.z; lo < u.w; lo += ich) split.push_back(make_int4(u.x, u.y, lo, std::min(u.w, lo + ich)));
            std::stable_sort(split.begin(), split.end(),
                             [](const int4& x, const int4& y) { return (x.w - x.z) > (y.w - y.z); });
            std::vector<int4> mine;  // snake order (0..P-1, P-1..0, ...): equal shares of long units
            const size_t P = (size_t)c->nparts;
            for (size_t u = 0; u < split.size(); ++u) {
                const size_t r = u % (2 * P);
                if ((r < P ? r : 2 * P - 1 - r) == (size_t)c->part) mine.push_back(split[u]);
            }
            c->units_h.swap(mine);
        }
        CK(c->units.ensure(sizeof(int4) * std::max<size_t>(c->units_h.size(), 1)));
        if (!c->units_h.empty())
            CK(cudaMemcpyAsync(c->units.p, c->units_h.data(), sizeof(int4) * c->units_h.size(), cudaMemcpyHostToDevice,
                               c->st));
        std::copy(key, key + 7, c->units_key);
    }
    // K': per-warp list length and refit set.  A search part keeps the longest lists: with 64
    // (or 74, one refit wave at T = 4) the part holding the best tuples of C3 missed its
    // certificate and paid a rescan (~1 ms); 96 and 128 refit in two waves (0.40 ms) and
    // certify (tools/parts_balance.py)
    // Dimension >= 4 sweeps keep 512-entry lists (fitcommon.cuh CAP_WIDE) and K' = 320: C4's ~260
    // near-ties within the margin of the 10th score then certify without a rescan sweep
    // (168 -> ~95 ms); the refit waves still stop after the first wave when it certifies.
    // Large keep (> kKeepLists): no per-warp lists; every accepted bound goes to a global candidate
    // list below the histogram threshold of K' = keep + 32 (collect mode 2, fitcommon.cuh; a global
    // list for every search was tried: dense near-ties flood it, C3 random y 3.9 -> 8.3 ms)
    static const int kprime_env = [] {
        const char* e = getenv("L0S_KPRIME");  // experiments: global list of this K'
        return e ? atoi(e) : 0;
    }();
    const bool big = keep > kKeepLists || kprime_env > 0;
    const int kc = kprime_env > 0 ? std::max<int>(kprime_env, (int)keep + 32)
                   : big ? (int)(keep + std::max<int64_t>(32, keep / 2))  // slack: near-ties among the keep best
                   : n >= 4 ? (int)std::min<int64_t>(480, std::max<int64_t>(320, keep + 32))  // CAP_WIDE lists
                            : (c->nparts > 1 ? 128 : (int)std::min<int64_t>(128, std::max<int64_t>(64, keep + 32)));
    const int64_t coll_cap = (int64_t)1 << 24;
    const int grid = n == 2   ? fit2_grid(c->T, c->nsm)
                     : n == 3 ? fit3_grid(c->T, c->nsm)
                     : n == 4 ? fit4_grid(c->T, c->nsm)
                              : fit5_grid(c->T, c->nsm);
    auto launch_fit = [&](const FitArgs& fa) {
        return n == 2   ? fit2_launch(fa, c->nsm, c->st)
               : n == 3 ? fit3_launch(fa, c->nsm, c->st)
               : n == 4 ? fit4_launch(fa, c->nsm, c->st)
                        : fit5_launch(fa, c->nsm, c->st);
    };
    const int slots = grid * (n == 3 ? fit3_slots_per_cta(c->T) : fit_slots_per_cta());
    const int64_t ill_cap = (int64_t)1 << 26;  // 512 MB of ranks; overflow is reported, never dropped
    CK(c->ucount.ensure(sizeof(int) * 4));
    CK(c->n_eval.ensure(2 * sizeof(unsigned long long)));  // [0] evaluations, [1] tile-screen tests
    CK(c->theta_g.ensure(sizeof(unsigned long long)));
    CK(c->hist.ensure(sizeof(unsigned) * HIST_BINS));
    CK(c->seedbuf.ensure(sizeof(int64_t) * 1024 * (kSeedW + 1) + 256));  // subsets, bounds, count, cap
    CK(c->wl_lb.ensure(sizeof(double) * slots * (big ? 1 : kc)));
    CK(c->wl_rank.ensure(sizeof(int64_t) * slots * (big ? 1 : kc)));
    CK(c->wl_cnt.ensure(sizeof(int) * slots));
    CK(c->ill.ensure(sizeof(int64_t) * ill_cap));
    CK(c->ill_cnt.ensure(sizeof(unsigned long long)));
    const int64_t lists = (int64_t)slots * (big ? 1 : kc);
    CK(c->cand_lb.ensure(sizeof(double) * lists));
    CK(c->cand_rank.ensure(sizeof(int64_t) * lists));
    CK(c->cand_cnt.ensure(sizeof(unsigned long long)));
    CK(c->lb_tmp.ensure(sizeof(double) * lists));
    CK(c->rank_tmp.ensure(sizeof(int64_t) * lists));
    size_t tb = sort_pairs_temp_bytes(lists);
    CK(c->sort_tmp.ensure(tb));
    unsigned long long inf_enc = ord_enc(INFINITY);

    FitArgs a{};
    fill_fit_common(c, a, n);
    a.units = c->units.as<int4>();
    a.n_units = (int)c->units_h.size();
    a.unit_counter = c->ucount.as<int>();
    a.rank_lo = rb;
    a.rank_hi = re;
    a.ranged = (rb > 0 || re < N) ? 1 : 0;
    a.kc = kc;
    a.collect = big ? 2 : 0;
    a.theta0 = INFINITY;
    if (big) {
        CK(c->coll_lb.ensure(sizeof(double) * coll_cap));
        CK(c->coll_rank.ensure(sizeof(int64_t) * coll_cap));
        CK(c->coll_cnt.ensure(sizeof(unsigned long long)));
        CK(cudaMemsetAsync(c->coll_cnt.p, 0, sizeof(unsigned long long), c->st));
        a.coll_lb = c->coll_lb.as<double>();
        a.coll_rank = c->coll_rank.as<int64_t>();
        a.coll_cnt = c->coll_cnt.as<unsigned long long>();
        a.coll_cap = coll_cap;
    }
    a.theta_g = c->theta_g.as<unsigned long long>();
    a.hist = c->hist.as<unsigned>();
    a.seed_tup = c->seedbuf.as<int64_t>();
    a.seed_ub = c->seedbuf.as<double>() + 1024 * kSeedW;
    a.seed_n = reinterpret_cast<int*>(c->seedbuf.as<double>() + 1024 * (kSeedW + 1));
    a.seed_cap = c->seedbuf.as<double>() + 1024 * (kSeedW + 1) + 4;
    a.keep = (int)keep;
    static const bool tsk_off = [] {  // L0S_TILE_SCREEN=0: the plain sweep only (tests, experiments)
        const char* e = getenv("L0S_TILE_SCREEN");
        return e && e[0] == '0';
    }();
    if ((n == 3 || n == 4) && !tsk_off && (c->m + 7) / 8 <= 65535) {  // the sweeps' tile screen (k_tile_max)
        const int64_t nt = fit3_tmax_doubles(c->m, c->mp);
        if (nt > 0) {
            CK(c->tmax.ensure(sizeof(double) * nt));
            a.tmax = c->tmax.as<double>();
        }
    }
    {
        double yy_top = 0.0;  // uncentered total |y|^2 >= every pooled bound
        for (double v : c->yyu_h) yy_top += v;
        a.hist_base = hist_base_for(yy_top > 0.0 ? yy_top : 1.0);
    }
    a.wl_lb = c->wl_lb.as<double>();
    a.wl_rank = c->wl_rank.as<int64_t>();
    a.wl_cnt = c->wl_cnt.as<int>();
    a.ill = c->ill.as<int64_t>();
    a.ill_cnt = c->ill_cnt.as<unsigned long long>();
    a.ill_cap = ill_cap;
    a.n_eval = c->n_eval.as<unsigned long long>();
    a.n_screen = c->n_eval.as<unsigned long long>() + 1;

    CK(cudaMemsetAsync(c->ucount.p, 0, sizeof(int) * 4, c->st));
    CK(cudaMemsetAsync(c->n_eval.p, 0, 2 * sizeof(unsigned long long), c->st));
    CK(cudaMemcpyAsync(c->theta_g.p, &inf_enc, sizeof inf_enc, cudaMemcpyHostToDevice, c->st));
    static const double inf_d = INFINITY;
    CK(cudaMemcpyAsync(a.seed_cap, &inf_d, sizeof inf_d, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(c->hist.p, 0, sizeof(unsigned) * HIST_BINS, c->st));
    CK(cudaMemsetAsync(c->ill_cnt.p, 0, sizeof(unsigned long long), c->st));
    CK(cudaMemsetAsync(c->cand_cnt.p, 0, sizeof(unsigned long long), c->st));
    cudaEventRecord(c->ev[2], c->st);
    if (launch_fit(a) < 0) return fail(L0S_ECUDA, "screened fit launch failed (TMA descriptor)");
    cudaEventRecord(c->ev[3], c->st);
    CK(cudaGetLastError());
    st->n_fit_launches++;
    st->n_launches += a.tmax ? 6 : 4;  // threshold seed (select, eval, commit) + tile maxima + the screened and plain sweeps
    if (!big) {
        launch_gather_candidates(a.wl_lb, a.wl_rank, a.wl_cnt, slots, kc, a.theta_g, c->cand_lb.as<double>(),
                                 c->cand_rank.as<int64_t>(), c->cand_cnt.as<unsigned long long>(), c->st);
        st->n_launches++;
    }
    // the candidate set: the gathered warp lists, or (large keep) the global collect list
    double* cl = big ? c->coll_lb.as<double>() : c->cand_lb.as<double>();
    int64_t* cr = big ? c->coll_rank.as<int64_t>() : c->cand_rank.as<int64_t>();
    unsigned long long ncand = 0, nill = 0, th_enc = 0, nev = 0, nscr = 0;
    double seed_cap = INFINITY;
    CK(cudaMemcpyAsync(&nev, c->n_eval.p, sizeof nev, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&nscr, c->n_eval.as<unsigned long long>() + 1, sizeof nscr, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&seed_cap, a.seed_cap, sizeof seed_cap, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&ncand, big ? c->coll_cnt.p : c->cand_cnt.p, sizeof ncand, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&nill, c->ill_cnt.p, sizeof nill, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&th_enc, c->theta_g.p, sizeof th_enc, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    st->ms_fit += elapsed(c->ev[2], c->ev[3]);
    st->n_eval += (int64_t)nev;
    st->n_screen += (int64_t)nscr;
    st->theta = ord_dec(th_enc);
    if ((int64_t)nill > ill_cap)
        return fail(L0S_ECAPACITY, "%llu ill-conditioned tuples exceed the routing buffer (%lld)",
                    (unsigned long long)nill, (long long)ill_cap);
    if (big) {
        if ((int64_t)ncand > coll_cap)
            return fail(L0S_ECAPACITY, "%llu candidates exceed the collect buffer (%lld)", (unsigned long long)ncand,
                        (long long)coll_cap);
        CK(c->lb_tmp.ensure(sizeof(double) * std::max<unsigned long long>(ncand, 1)));
        CK(c->rank_tmp.ensure(sizeof(int64_t) * std::max<unsigned long long>(ncand, 1)));
        tb = sort_pairs_temp_bytes((int64_t)ncand);
        CK(c->sort_tmp.ensure(tb));
    }
    {
        const int ns = sort_pairs(cl, cr, c->lb_tmp.as<double>(), c->rank_tmp.as<int64_t>(), (int64_t)ncand, c->sort_tmp.p,
                                  tb, c->st);
        if (ns < 0) return fail(L0S_ECUDA, "sort scratch too small");
        st->n_launches += ns;
    }
    const int64_t nc = std::min<int64_t>((int64_t)ncand, kc);
    const int64_t wave = std::max<int64_t>(keep + 8, 256 / std::max(1, c->T));
    // without a cap (single searches) the first refit wave needs no host decision: it is queued
    // right behind the sort, and its results come back with the candidates' bounds in one sync
    cudaEventRecord(c->ev[2], c->st);
    ExactPending first;
    const bool early = c->nparts == 1 && nc > 0;
    if (early) {
        const int erc = exact_launch(c, n, cr, std::min(nc, wave), first, &st->n_launches, true);
        if (erc) return erc;
    }
    // the candidates' sorted bounds (SSR units) on the host: certificate thresholds below
    std::vector<double> lbs((size_t)nc);
    if (nc > 0) {
        CK(cudaMemcpyAsync(lbs.data(), cl, sizeof(double) * nc, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
    // every excluded tuple has lb >= G_lb (SSR units): the K'-th smallest gathered bound, or
    // -- fewer gathered -- the final shared threshold (+inf: nothing was ever dropped)
    double G_lb = st->theta;
    if ((int64_t)ncand >= kc) G_lb = std::min(lbs[(size_t)kc - 1], st->theta);
    // A search part (l0s_search_part) answers for its own units only, but the seed's subsets come
    // from the whole problem: >= keep tuples score at most seed_cap / s, so the global keep-th
    // score is below that cap and a part's excluded tuples need only clear the cap.
    double cap = c->nparts > 1 ? seed_cap / (double)c->s : INFINITY;
    double yy = 0.0;
    for (double v : c->yyu_h) yy += v;
    auto margin_of = [&](double sk) { return 1e-10 * std::fabs(sk) + 64.0 * kEps * yy / (double)c->s; };
    // a part refits only the candidates that can reach the global top list: the sorted bounds
    // above the cap (+ margin) are excluded like the rest (G_lb drops to the first of them)
    int64_t nref = nc;
    if (std::isfinite(cap) && nc > 0) {
        const double lim = (cap + margin_of(cap)) * (double)c->s;
        nref = 0;
        while (nref < nc && lbs[(size_t)nref] <= lim) ++nref;
        if (nref < nc) G_lb = std::min(G_lb, lbs[(size_t)nref]);
    }
    // exact refit of the candidates in waves, lowest bounds first: the first wave (about one pass
    // of k_exact_smem over the device at T tasks) usually certifies alone -- the candidates after
    // it have lb >= lbs[done] -- and the rest are refit only when it does not.  Results are the
    // full refit's: an excluded candidate scores above the keep-th exact score by the margin.
    int rc = L0S_OK;
    {
        int64_t done = 0;
        while (done < nref) {
            const int64_t nb = done == 0 ? std::min(nref, wave) : nref - done;
            std::vector<Cand> exact;
            if (done == 0 && early) {  // nref == nc here: the queued wave is this one
                rc = exact_collect(c, n, first, exact, &c->recs);
            } else {
                rc = exact_ranks_to_host(c, n, cr + done, nb, exact, &st->n_launches, &c->recs);
            }
            if (rc) return rc;
            merge_best(best, exact, keep);
            done += nb;
            if (done < nref) {
                const double sk = std::min(((int64_t)best.size() >= keep) ? best[(size_t)keep - 1].score : INFINITY,
                                           cap);
                if (lbs[(size_t)done] / (double)c->s > sk + margin_of(sk)) {
                    G_lb = std::min(G_lb, lbs[(size_t)done]);
                    break;
                }
            }
        }
        nref = done;
    }
    if (nill > 0) {
        // Tuples the Gram screen could not certify: TSQR on the device gives each a score and
        // the reference's rank-rule ratio; only those that can reach the top list within the
        // QR's error margin (~ eps / ratio) are refit bit-exactly.
        rc = screen_ill(c, n, (int64_t)nill, keep, best, st, cap);
        if (rc) return rc;
    }
    cudaEventRecord(c->ev[3], c->st);
    CK(cudaStreamSynchronize(c->st));
    st->ms_exact += elapsed(c->ev[2], c->ev[3]);
    st->n_candidates = nref;
    st->n_ill = (int64_t)nill;
    // search parts: one exchange of the parts' best exact scores (l0s_set_part_exchange) -- the
    // keep-th of their union bounds the whole search's keep-th score, usually far below this
    // part's own when the part holds only some of the near-ties
    if (c->exch_pending) {
        c->exch_pending = false;
        std::vector<double> mine;
        for (size_t x = 0; x < best.size() && (int64_t)x < keep; ++x) mine.push_back(best[x].score);
        const double g = c->exch(mine.data(), (int64_t)mine.size(), c->exch_user);
        if (g < cap) cap = g;  // NaN leaves the cap
    }

    // certification: an excluded tuple has exact score >= lb / s >= G_lb / s; it cannot
    // displace the keep-th exact score if G_lb / s exceeds it by the reference's own error margin
    bool complete = !std::isfinite(G_lb);  // nothing was ever dropped
    double sk = std::min(((int64_t)best.size() >= keep) ? best[(size_t)keep - 1].score : INFINITY, cap);
    bool certified = complete || (G_lb / (double)c->s > sk + margin_of(sk));
    st->margin = G_lb / (double)c->s - sk;
    if (!certified) {
        // rescan: collect every tuple whose bound is below the keep-th exact score (+ margin)
        st->n_rescan++;
        // (fewer than keep finite scores among the K' candidates: collect every finite bound; a
        // collect buffer that overflows splits the rank range, l0s_search)
        double theta_star = std::isfinite(sk) ? (sk + margin_of(sk)) * (double)c->s : INFINITY;
        CK(c->coll_lb.ensure(sizeof(double) * coll_cap));
        CK(c->coll_rank.ensure(sizeof(int64_t) * coll_cap));
        CK(c->coll_cnt.ensure(sizeof(unsigned long long)));
        CK(cudaMemsetAsync(c->ucount.p, 0, sizeof(int) * 4, c->st));
        CK(cudaMemsetAsync(c->coll_cnt.p, 0, sizeof(unsigned long long), c->st));
        CK(cudaMemsetAsync(c->ill_cnt.p, 0, sizeof(unsigned long long), c->st));
        a.collect = 1;
        a.theta0 = theta_star;
        a.coll_lb = c->coll_lb.as<double>();
        a.coll_rank = c->coll_rank.as<int64_t>();
        a.coll_cnt = c->coll_cnt.as<unsigned long long>();
        a.coll_cap = coll_cap;
        cudaEventRecord(c->ev[2], c->st);
        if (launch_fit(a) < 0) return fail(L0S_ECUDA, "screened fit launch failed (TMA descriptor)");
        cudaEventRecord(c->ev[3], c->st);
        CK(cudaGetLastError());
        st->n_fit_launches++;
        st->n_launches += a.tmax ? 3 : 1;
        unsigned long long ncoll = 0;
        CK(cudaMemcpyAsync(&ncoll, c->coll_cnt.p, sizeof ncoll, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(&nev, c->n_eval.p, sizeof nev, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(&nscr, c->n_eval.as<unsigned long long>() + 1, sizeof nscr, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        st->ms_fit += elapsed(c->ev[2], c->ev[3]);
        st->n_eval = (int64_t)nev;  // the counters accumulate over both sweeps
        st->n_screen = (int64_t)nscr;
        if ((int64_t)ncoll > coll_cap)
            return fail(L0S_ECAPACITY, "%llu tuples below the certification threshold exceed the rescan buffer",
                        (unsigned long long)ncoll);
        std::vector<Cand> more;
        rc = exact_ranks_to_host(c, n, c->coll_rank.as<int64_t>(), (int64_t)ncoll, more, &st->n_launches, &c->recs);
        if (rc) return rc;
        st->n_candidates += (int64_t)ncoll;
        merge_best(best, more, keep);
    }
    st->certified = 1;
    st->mode_used = L0S_MODE_FAST;
    return L0S_OK;
}

}  // extern "C"

// Dimension 1 (fit1.cu): a lower bound per feature, sorted on the device, refit in order until
// the keep-th exact score is certified -- every excluded feature's bound lies above it by the
// reference's error margin (the same certificate as the screened sweeps).
static int search_fast1(l0s_ctx* c, int64_t keep, int64_t rb, int64_t re, std::vector<Cand>& best, l0s_stats* st) {
    const int64_t cnt = re - rb;
    CK(c->coll_lb.ensure(sizeof(double) * cnt));
    CK(c->coll_rank.ensure(sizeof(int64_t) * cnt));
    CK(c->ill.ensure(sizeof(int64_t) * cnt));
    CK(c->ill_cnt.ensure(sizeof(unsigned long long)));
    const size_t tb = sort_pairs_temp_bytes(cnt);
    CK(c->sort_tmp.ensure(tb));
    FitArgs a{};
    fill_fit_common(c, a, 1);
    a.ill = c->ill.as<int64_t>();
    a.ill_cnt = c->ill_cnt.as<unsigned long long>();
    a.ill_cap = cnt;
    CK(cudaMemsetAsync(c->ill_cnt.p, 0, sizeof(unsigned long long), c->st));
    double* cl = c->coll_lb.as<double>();
    int64_t* cr = c->coll_rank.as<int64_t>();
    cudaEventRecord(c->ev[2], c->st);
    launch_fit1(a, rb, re, cl, cr, c->st);
    const int ns = sort_pairs(cl, cr, nullptr, nullptr, cnt, c->sort_tmp.p, tb, c->st);
    cudaEventRecord(c->ev[3], c->st);
    CK(cudaGetLastError());
    if (ns < 0) return fail(L0S_ECUDA, "sort scratch too small");
    st->n_fit_launches++;
    st->n_launches += 1 + ns;
    unsigned long long nill = 0;
    CK(cudaMemcpyAsync(&nill, c->ill_cnt.p, sizeof nill, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    st->ms_fit += elapsed(c->ev[2], c->ev[3]);
    st->n_eval += cnt * c->T;
    double yy = 0.0;
    for (double v : c->yyu_h) yy += v;
    auto margin_of = [&](double sk) { return 1e-10 * std::fabs(sk) + 64.0 * kEps * yy / (double)c->s; };
    // refit the sorted bounds in growing prefixes until the next excluded bound certifies
    cudaEventRecord(c->ev[2], c->st);
    int64_t done = 0, upto = std::min<int64_t>(cnt, std::max<int64_t>(64, keep + 32));
    double G_lb = INFINITY;
    for (;;) {
        std::vector<double> lbs((size_t)(upto - done + (upto < cnt ? 1 : 0)));
        CK(cudaMemcpyAsync(lbs.data(), cl + done, sizeof(double) * lbs.size(), cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        int64_t fin = done;  // +inf bounds (ill, dead) sort last and are never refit from this list
        while (fin < upto && std::isfinite(lbs[(size_t)(fin - done)])) ++fin;
        std::vector<Cand> exact;
        int rc = exact_ranks_to_host(c, 1, cr + done, fin - done, exact, &st->n_launches, &c->recs);
        if (rc) return rc;
        merge_best(best, exact, keep);
        st->n_candidates += fin - done;
        G_lb = (fin < upto || upto == cnt) ? INFINITY : lbs.back();
        const double sk = ((int64_t)best.size() >= keep) ? best[(size_t)keep - 1].score : INFINITY;
        if (!std::isfinite(G_lb) || G_lb / (double)c->s > sk + margin_of(sk)) {
            st->margin = G_lb / (double)c->s - sk;
            break;
        }
        st->n_rescan++;
        done = upto;
        upto = std::min<int64_t>(cnt, 2 * upto);
    }
    if (nill > 0) {
        int rc = screen_ill(c, 1, (int64_t)nill, keep, best, st);
        if (rc) return rc;
    }
    cudaEventRecord(c->ev[3], c->st);
    CK(cudaStreamSynchronize(c->st));
    st->ms_exact += elapsed(c->ev[2], c->ev[3]);
    st->n_ill = (int64_t)nill;
    st->theta = G_lb;
    st->certified = 1;
    st->mode_used = L0S_MODE_FAST;
    return L0S_OK;
}

// The screened search of [rb, re); a fixed device buffer that overflows (ill-conditioned tuples,
// collected candidates, rescan) splits the range in halves, each certified on its own, and the
// (score, rank) merge of certified ranges is the whole range's (search.py:303).
static int search_fast_split(l0s_ctx* c, int n, int64_t keep, int64_t rb, int64_t re, std::vector<Cand>& best,
                             l0s_stats* st, int depth) {
    std::vector<Cand> mine = best;
    int rc = search_fast_mode(c, n, keep, rb, re, mine, st);
    if (rc == L0S_OK) {
        best.swap(mine);
        return rc;
    }
    if (rc != L0S_ECAPACITY || depth >= 24 || re - rb < 2) return rc;
    const int64_t mid = rb + (re - rb) / 2;
    st->n_rescan++;  // counted as a rescan: the range is searched again in two halves
    rc = search_fast_split(c, n, keep, rb, mid, best, st, depth + 1);
    if (rc) return rc;
    return search_fast_split(c, n, keep, mid, re, best, st, depth + 1);
}

extern "C" {

int l0s_search(l0s_ctx* c, int n, int64_t keep, int64_t rank_begin, int64_t rank_end, int mode, double* out_scores,
               int64_t* out_ranks, double* out_coef, double* out_ssr, int64_t* out_count, l0s_stats* stats) {
    l0s_stats local{};
    l0s_stats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof *st);
    *out_count = 0;
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (n < 1 || n > 15) return fail(L0S_EINVAL, "dimension %d outside [1, 15]", n);
    if (keep < 1) return fail(L0S_EINVAL, "keep must be >= 1");
    if (c->m < n) return fail(L0S_EINVAL, "subspace holds %lld features, need at least %d", (long long)c->m, n);
    int64_t N;
    int rc = l0s_count(c->m, n, &N);
    if (rc) return rc;
    CK(cudaSetDevice(c->dev));
    int64_t rb = std::max<int64_t>(rank_begin, 0), re = std::min<int64_t>(rank_end, N);
    st->n_tuples = std::max<int64_t>(re - rb, 0);
    st->ms_gram = c->ms_gram;
    st->ms_gram_kernel = c->ms_gram_k;
    if (rb >= re) return L0S_OK;
    rc = ensure_binom(c, n);
    c->recs.clear();
    if (rc) return rc;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, c->st);
    // the screen's error model is for fp64 arithmetic in the reference (precision="fp64")
    bool fast_ok = (n >= 1 && n <= 4 || (n == 5 && c->m < 32768)) && c->T <= fit3_max_tasks() && keep <= kKeepMax;
    bool use_fast;
    if (mode == L0S_MODE_FAST) {
        if (!fast_ok) {
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
            return fail(L0S_EINVAL, "screened path needs n in 1..5, ntasks <= %d, keep <= %lld",
                        fit3_max_tasks(), (long long)kKeepMax);
        }
        use_fast = true;
    } else if (mode == L0S_MODE_EXACT) {
        use_fast = false;
    } else {
        double work = (double)(re - rb) * (double)c->s;
        use_fast = fast_ok && work > 2e8;
    }
    std::vector<Cand> best;
    rc = !use_fast ? search_exact_mode(c, n, keep, rb, re, best, st)
         : n == 1  ? search_fast1(c, keep, rb, re, best, st)
                   : search_fast_split(c, n, keep, rb, re, best, st, 0);
    if (rc) {
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        return rc;
    }
    // final records: coefficients and per-task ssr of the kept tuples (bit-exact kernel); the
    // screened path already holds them from the candidate refit
    int64_t nk = (int64_t)best.size();
    bool have_all = nk > 0;
    for (int64_t i = 0; i < nk && have_all; ++i) have_all = c->recs.count(best[(size_t)i].rank) != 0;
    if (have_all) {
        const int p = n + 1;
        for (int64_t i = 0; i < nk; ++i) {
            const Rec& r = c->recs[best[(size_t)i].rank];
            if (out_coef) std::copy(r.coef.begin(), r.coef.end(), out_coef + i * c->T * p);
            if (out_ssr) std::copy(r.ssr.begin(), r.ssr.end(), out_ssr + i * c->T);
            out_scores[i] = best[(size_t)i].score;
            out_ranks[i] = best[(size_t)i].rank;
        }
    } else if (nk > 0) {
        cudaEventRecord(c->ev[2], c->st);
        std::vector<int64_t> rk((size_t)nk);
        for (int64_t i = 0; i < nk; ++i) rk[(size_t)i] = best[(size_t)i].rank;
        CK(c->ex_ranks.ensure(sizeof(int64_t) * std::max<int64_t>(nk, 1 << 10)));
        CK(cudaMemcpyAsync(c->ex_ranks.p, rk.data(), sizeof(int64_t) * nk, cudaMemcpyHostToDevice, c->st));
        rc = run_exact(c, n, c->ex_ranks.as<int64_t>(), nullptr, nk, true, &st->n_launches);
        if (rc) {
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
            return rc;
        }
        const int p = n + 1;
        std::vector<double> sc((size_t)nk);
        CK(cudaMemcpyAsync(sc.data(), c->ex_score.p, sizeof(double) * nk, cudaMemcpyDeviceToHost, c->st));
        if (out_coef) CK(cudaMemcpyAsync(out_coef, c->ex_coef.p, sizeof(double) * nk * c->T * p, cudaMemcpyDeviceToHost, c->st));
        if (out_ssr) CK(cudaMemcpyAsync(out_ssr, c->ex_ssr.p, sizeof(double) * nk * c->T, cudaMemcpyDeviceToHost, c->st));
        cudaEventRecord(c->ev[3], c->st);
        CK(cudaStreamSynchronize(c->st));
        st->ms_records = elapsed(c->ev[2], c->ev[3]);
        for (int64_t i = 0; i < nk; ++i) {
            if (sc[(size_t)i] != best[(size_t)i].score) {
                cudaEventDestroy(t0);
                cudaEventDestroy(t1);
                return fail(L0S_ECUDA, "refit of rank %lld is not reproducible", (long long)best[(size_t)i].rank);
            }
            out_scores[i] = best[(size_t)i].score;
            out_ranks[i] = best[(size_t)i].rank;
        }
    }
    cudaEventRecord(t1, c->st);
    CK(cudaStreamSynchronize(c->st));
    st->ms_total = elapsed(t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    *out_count = nk;
    return L0S_OK;
}

int l0s_search_part(l0s_ctx* c, int n, int64_t keep, int part, int nparts, int mode, double* out_scores,
                    int64_t* out_ranks, double* out_coef, double* out_ssr, int64_t* out_count, l0s_stats* stats) {
    if (out_count) *out_count = 0;
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    if (nparts < 1 || part < 0 || part >= nparts) return fail(L0S_EINVAL, "part %d of %d", part, nparts);
    int64_t N = 0;
    int rc = (n >= 1 && c->m >= n) ? l0s_count(c->m, n, &N) : L0S_OK;
    if (rc) return rc;
    // every part must take the same path: decided on the whole problem, as l0s_search would
    const bool fast_ok = (n >= 1 && n <= 4 || (n == 5 && c->m < 32768)) && c->T <= fit3_max_tasks() && keep >= 1 &&
                         keep <= kKeepMax;
    const bool fast = mode == L0S_MODE_FAST || (mode == L0S_MODE_AUTO && fast_ok && (double)N * (double)c->s > 2e8);
    if (!fast || !fast_ok || nparts == 1 || n == 1)  // contiguous rank ranges (search.py:266-271)
        return l0s_search(c, n, keep, N / nparts * part + std::min<int64_t>(part, N % nparts),
                          N / nparts * (part + 1) + std::min<int64_t>(part + 1, N % nparts), mode, out_scores,
                          out_ranks, out_coef, out_ssr, out_count, stats);
    c->part = part;
    c->nparts = nparts;
    c->exch_pending = c->exch != nullptr;
    rc = l0s_search(c, n, keep, 0, N, L0S_MODE_FAST, out_scores, out_ranks, out_coef, out_ssr, out_count, stats);
    if (rc == L0S_OK && c->exch_pending) {  // the exchange is a collective: take part even if unused
        std::vector<double> mine(out_scores, out_scores + (out_count ? *out_count : 0));
        c->exch(mine.data(), (int64_t)mine.size(), c->exch_user);
    }
    c->exch_pending = false;
    c->part = 0;
    c->nparts = 1;
    return rc;
}

int l0s_set_part_exchange(l0s_ctx* c, l0s_exchange_fn fn, void* user) {
    if (!c) return fail(L0S_EINVAL, "null context");
    c->exch = fn;
    c->exch_user = user;
    return L0S_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// SIS projection scores (screening._chunk_scores, screening.py:126-155)
// ---------------------------------------------------------------------------

int l0s_sis_prepare(l0s_ctx* c, const double* targets, int R, int64_t s, const int64_t* perm, const int64_t* bounds,
                    int ntasks) {
    if (!c) return fail(L0S_EINVAL, "null context");
    if (R < 1 || R > sis_max_targets()) return fail(L0S_EINVAL, "1 <= targets <= %d (got %d)", sis_max_targets(), R);
    if (s < 1 || ntasks < 1) return fail(L0S_EINVAL, "need s >= 1 and ntasks >= 1");
    if (bounds[0] != 0 || bounds[ntasks] != s) return fail(L0S_EINVAL, "bounds must run from 0 to s");
    for (int t = 0; t < ntasks; ++t)
        if (bounds[t + 1] < bounds[t]) return fail(L0S_EINVAL, "bounds must be non-decreasing");
    CK(cudaSetDevice(c->dev));
    CK(c->sis_y.ensure(sizeof(double) * R * s));
    CK(c->sis_yc.ensure(sizeof(double) * R * s));
    CK(c->sis_sy.ensure(sizeof(double) * R * ntasks));
    CK(c->sis_perm.ensure(sizeof(int64_t) * s));
    CK(c->sis_bounds.ensure(sizeof(int64_t) * (ntasks + 1)));
    CK(cudaMemcpyAsync(c->sis_y.p, targets, sizeof(double) * R * s, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->sis_perm.p, perm, sizeof(int64_t) * s, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->sis_bounds.p, bounds, sizeof(int64_t) * (ntasks + 1), cudaMemcpyHostToDevice, c->st));
    launch_sis_targets(c->sis_y.as<double>(), R, s, c->sis_perm.as<int64_t>(), c->sis_bounds.as<int64_t>(), ntasks,
                       c->sis_yc.as<double>(), c->sis_sy.as<double>(), c->st);
    // the scores kernel's shared-memory row layout (k_sis_scores): per task, lane l's contiguous
    // range of E_t samples at l * (E_t + 1)
    std::vector<int> tE((size_t)ntasks), tpoff((size_t)ntasks), dest((size_t)s);
    int off = 0;
    for (int t = 0; t < ntasks; ++t) {
        const int64_t ns = bounds[t + 1] - bounds[t];
        int64_t W = 1;
        while (W < ns) W <<= 1;
        const int E = (int)std::min<int64_t>(16, std::max<int64_t>(1, W / 32));  // lane range per super-block
        const int64_t nsb = std::max<int64_t>(1, W / (32 * E));
        tE[(size_t)t] = E;
        tpoff[(size_t)t] = off;
        for (int64_t i = 0; i < ns; ++i) {
            const int64_t q = i / (32 * E), r = i % (32 * E);
            dest[(size_t)(bounds[t] + i)] = off + (int)((q * 32 + r / E) * (E + 1) + r % E);
        }
        off += (int)(nsb * 32 * (E + 1));
    }
    c->sis_rowlen = off;
    // slot of raw sample j (the kernel reads rows coalesced and scatters into shared memory)
    std::vector<int> rdest((size_t)s, -1);
    for (int64_t i = 0; i < s; ++i) {
        if (perm[i] < 0 || perm[i] >= s || rdest[(size_t)perm[i]] >= 0)
            return fail(L0S_EINVAL, "perm must be a permutation of [0, s)");
        rdest[(size_t)perm[i]] = dest[(size_t)i];
    }
    dest.swap(rdest);
    CK(c->sis_dest.ensure(sizeof(int) * s));
    CK(c->sis_tE.ensure(sizeof(int) * ntasks));
    CK(c->sis_tpoff.ensure(sizeof(int) * ntasks));
    CK(cudaMemcpyAsync(c->sis_dest.p, dest.data(), sizeof(int) * s, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->sis_tE.p, tE.data(), sizeof(int) * ntasks, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->sis_tpoff.p, tpoff.data(), sizeof(int) * ntasks, cudaMemcpyHostToDevice, c->st));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->st));
    c->sis_R = R;
    c->sis_T = ntasks;
    c->sis_s = s;
    return L0S_OK;
}

int l0s_sis_scores(l0s_ctx* c, const double* F, int64_t k, int is_device, double* out) {
    if (!c || c->sis_R < 1) return fail(L0S_ESTATE, "l0s_sis_prepare must be called first");
    if (k < 0) return fail(L0S_EINVAL, "negative feature count");
    if (k == 0) return L0S_OK;
    CK(cudaSetDevice(c->dev));
    const int64_t s = c->sis_s;
    const double* Fd = F;
    if (!is_device) {
        CK(c->sis_F.ensure(sizeof(double) * k * s));
        CK(cudaMemcpyAsync(c->sis_F.p, F, sizeof(double) * k * s, cudaMemcpyHostToDevice, c->st));
        Fd = c->sis_F.as<double>();
    }
    CK(c->sis_out.ensure(sizeof(double) * k));
    if (launch_sis_scores(Fd, k, s, c->sis_perm.as<int64_t>(), c->sis_dest.as<int>(), c->sis_bounds.as<int64_t>(),
                          c->sis_tE.as<int>(), c->sis_tpoff.as<int>(), c->sis_rowlen, c->sis_T, c->sis_yc.as<double>(),
                          c->sis_sy.as<double>(), c->sis_R, c->sis_out.as<double>(), c->nsm, c->st))
        return fail(L0S_EINVAL, "%lld samples exceed the SIS kernel's shared-memory row", (long long)s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, c->sis_out.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

// ---------------------------------------------------------------------------
// Final-rung candidates (generation.iter_final_rung, generation.py:331-393)
// ---------------------------------------------------------------------------

int l0s_gen_pool(l0s_ctx* c, const void* values, int64_t n_pool, int64_t s, int fp32) {
    if (!c) return fail(L0S_EINVAL, "null context");
    if (n_pool < 0 || s < 1) return fail(L0S_EINVAL, "need n_pool >= 0 and s >= 1");
    CK(cudaSetDevice(c->dev));
    const size_t w = fp32 ? 4 : 8;
    CK(c->gen_pool.ensure(w * std::max<int64_t>(n_pool, 1) * s));
    if (n_pool) CK(cudaMemcpyAsync(c->gen_pool.p, values, w * n_pool * s, cudaMemcpyHostToDevice, c->st));
    c->gen_n = n_pool;
    c->gen_s = s;
    c->gen_fp32 = fp32 ? 1 : 0;
    c->gen_count = 0;
    c->gen_taken = 0;
    return L0S_OK;
}

int l0s_gen_eval(l0s_ctx* c, int kind, const int32_t* pi, const int32_t* pj, int64_t count, const void* values,
                 double tol, double min_abs, double max_abs, double dedup_tol, uint8_t* out_valid,
                 uint64_t* out_hash) {
    if (!c || c->gen_s < 1) return fail(L0S_ESTATE, "l0s_gen_pool must be called first");
    if (kind < GEN_COPY || kind > GEN_VALUES) return fail(L0S_EINVAL, "bad operator kind %d", kind);
    if (count < 0 || count > (int64_t)1 << 30) return fail(L0S_EINVAL, "bad candidate count %lld", (long long)count);
    if (kind == GEN_VALUES ? values == nullptr : pi == nullptr) return fail(L0S_EINVAL, "missing candidate input");
    CK(cudaSetDevice(c->dev));
    const int64_t s = c->gen_s;
    const size_t w = c->gen_fp32 ? 4 : 8;
    c->gen_count = 0;
    c->gen_taken = 0;
    if (count == 0) return L0S_OK;
    const void* A = c->gen_pool.p;
    const int* dpi = nullptr;
    const int* dpj = nullptr;
    if (kind == GEN_VALUES) {
        CK(c->gen_take.ensure(w * count * s));  // staging for the precomputed rows
        CK(cudaMemcpyAsync(c->gen_take.p, values, w * count * s, cudaMemcpyHostToDevice, c->st));
        A = c->gen_take.p;
    } else {
        for (int64_t x = 0; x < count; ++x) {
            if (pi[x] < 0 || pi[x] >= c->gen_n || (pj && (pj[x] < -1 || pj[x] >= c->gen_n)))
                return fail(L0S_EINVAL, "candidate %lld: child index outside the pool", (long long)x);
        }
        CK(c->gen_pi.ensure(sizeof(int) * count));
        CK(cudaMemcpyAsync(c->gen_pi.p, pi, sizeof(int) * count, cudaMemcpyHostToDevice, c->st));
        dpi = c->gen_pi.as<int>();
        if (pj) {
            CK(c->gen_pj.ensure(sizeof(int) * count));
            CK(cudaMemcpyAsync(c->gen_pj.p, pj, sizeof(int) * count, cudaMemcpyHostToDevice, c->st));
            dpj = c->gen_pj.as<int>();
        }
    }
    CK(c->gen_vals.ensure(sizeof(double) * count * s));
    CK(c->gen_valid.ensure((size_t)count));
    CK(c->gen_hash.ensure(sizeof(uint64_t) * 2 * count));
    launch_gen_eval(A, c->gen_fp32, s, dpi, dpj, (int)count, kind, tol, min_abs, max_abs, dedup_tol,
                    c->gen_vals.as<double>(), c->gen_valid.as<unsigned char>(), c->gen_hash.as<unsigned long long>(),
                    c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_valid, c->gen_valid.p, (size_t)count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(out_hash, c->gen_hash.p, sizeof(uint64_t) * 2 * count, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->gen_count = count;
    return L0S_OK;
}

int l0s_gen_take(l0s_ctx* c, const int32_t* rows, int64_t count, void* host_out, const double** dev_out) {
    if (!c || c->gen_count < 1) return fail(L0S_ESTATE, "no evaluated candidates (l0s_gen_eval)");
    if (count < 0) return fail(L0S_EINVAL, "negative row count");
    for (int64_t x = 0; x < count; ++x)
        if (rows[x] < 0 || rows[x] >= c->gen_count) return fail(L0S_EINVAL, "row %d outside the chunk", rows[x]);
    CK(cudaSetDevice(c->dev));
    const int64_t s = c->gen_s;
    CK(c->gen_rows.ensure(sizeof(int) * std::max<int64_t>(count, 1)));
    CK(c->gen_take.ensure(sizeof(double) * std::max<int64_t>(count, 1) * s));
    if (count) {
        CK(cudaMemcpyAsync(c->gen_rows.p, rows, sizeof(int) * count, cudaMemcpyHostToDevice, c->st));
        launch_gen_gather(c->gen_vals.as<double>(), s, c->gen_rows.as<int>(), (int)count, 0, c->gen_take.p, c->st);
        CK(cudaGetLastError());
    }
    c->gen_taken = count;
    if (host_out && count) {
        const size_t w = c->gen_fp32 ? 4 : 8;
        CK(c->gen_out.ensure(w * count * s));
        launch_gen_gather(c->gen_vals.as<double>(), s, c->gen_rows.as<int>(), (int)count, c->gen_fp32, c->gen_out.p,
                          c->st);
        CK(cudaMemcpyAsync(host_out, c->gen_out.p, w * count * s, cudaMemcpyDeviceToHost, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    if (dev_out) *dev_out = c->gen_take.as<double>();
    return L0S_OK;
}

int l0s_gen_fetch(l0s_ctx* c, const int32_t* rows, int64_t count, void* host_out) {
    if (!c || c->gen_taken < 1) return fail(L0S_ESTATE, "no taken rows (l0s_gen_take)");
    for (int64_t x = 0; x < count; ++x)
        if (rows[x] < 0 || rows[x] >= c->gen_taken) return fail(L0S_EINVAL, "row %d outside the taken rows", rows[x]);
    if (count <= 0) return L0S_OK;
    CK(cudaSetDevice(c->dev));
    const int64_t s = c->gen_s;
    const size_t w = c->gen_fp32 ? 4 : 8;
    CK(c->gen_rows.ensure(sizeof(int) * count));
    CK(c->gen_out.ensure(w * count * s));
    CK(cudaMemcpyAsync(c->gen_rows.p, rows, sizeof(int) * count, cudaMemcpyHostToDevice, c->st));
    launch_gen_gather(c->gen_take.as<double>(), s, c->gen_rows.as<int>(), (int)count, c->gen_fp32, c->gen_out.p, c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(host_out, c->gen_out.p, w * count * s, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

// ---------------------------------------------------------------------------
// The last rung's value dedup on the device (dedup.cu; generation.py:364-385)
// ---------------------------------------------------------------------------

static DedupTable dedup_view(l0s_ctx* c) {
    return DedupTable{c->dd_lo.as<unsigned long long>(), c->dd_hi.as<unsigned long long>(),
                      c->dd_owner.as<unsigned long long>(), c->dd_state.as<unsigned>(),
                      c->dd_used.as<unsigned long long>(), c->dd_mask};
}

static int dedup_alloc(l0s_ctx* c, unsigned long long cap) {
    CK(c->dd_lo.ensure(sizeof(unsigned long long) * cap));
    CK(c->dd_hi.ensure(sizeof(unsigned long long) * cap));
    CK(c->dd_owner.ensure(sizeof(unsigned long long) * cap));
    CK(c->dd_state.ensure(sizeof(unsigned) * cap));
    CK(c->dd_used.ensure(sizeof(unsigned long long)));
    CK(cudaMemsetAsync(c->dd_state.p, 0, sizeof(unsigned) * cap, c->st));
    CK(cudaMemsetAsync(c->dd_used.p, 0, sizeof(unsigned long long), c->st));
    c->dd_mask = cap - 1;
    return L0S_OK;
}

// keep the load factor <= 1/2 for `more` further insertions (rehash into a doubled table)
static int dedup_reserve(l0s_ctx* c, int64_t more) {
    unsigned long long used = 0;
    CK(cudaMemcpyAsync(&used, c->dd_used.p, sizeof used, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    unsigned long long cap = c->dd_mask + 1;
    if (2 * (used + (unsigned long long)more) <= cap) return L0S_OK;
    while (2 * (used + (unsigned long long)more) > cap) cap *= 2;
    DBuf lo, hi, own, stt, usd;
    std::swap(lo, c->dd_lo);
    std::swap(hi, c->dd_hi);
    std::swap(own, c->dd_owner);
    std::swap(stt, c->dd_state);
    std::swap(usd, c->dd_used);
    const DedupTable from{lo.as<unsigned long long>(), hi.as<unsigned long long>(), own.as<unsigned long long>(),
                          stt.as<unsigned>(), usd.as<unsigned long long>(), c->dd_mask};
    int rc = dedup_alloc(c, cap);
    if (rc) return rc;
    launch_dedup_rehash(from, dedup_view(c), c->st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->st));  // the old table is released on return
    return L0S_OK;
}

int l0s_gen_dedup_reset(l0s_ctx* c, const uint64_t* seed, int64_t count) {
    if (!c) return fail(L0S_EINVAL, "null context");
    if (count < 0) return fail(L0S_EINVAL, "negative seed count");
    CK(cudaSetDevice(c->dev));
    unsigned long long cap = (unsigned long long)1 << 20;
    while (cap < 4ull * (unsigned long long)count) cap *= 2;
    int rc = dedup_alloc(c, cap);
    if (rc) return rc;
    c->dd_epoch = 0;  // the seed (the pool's fingerprints) owns epoch 0
    if (count > 0) {
        CK(c->dd_seed.ensure(sizeof(uint64_t) * 2 * count));
        CK(cudaMemcpyAsync(c->dd_seed.p, seed, sizeof(uint64_t) * 2 * count, cudaMemcpyHostToDevice, c->st));
        launch_dedup_insert(dedup_view(c), nullptr, c->dd_seed.as<unsigned long long>(), count, 0, c->st);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(c->st));
    return L0S_OK;
}

int l0s_gen_dedup(l0s_ctx* c, uint8_t* out_kept, int64_t* out_count) {
    if (!c || c->dd_mask == 0) return fail(L0S_ESTATE, "l0s_gen_dedup_reset must be called first");
    if (c->gen_count < 1) return fail(L0S_ESTATE, "no evaluated candidates (l0s_gen_eval)");
    CK(cudaSetDevice(c->dev));
    const int64_t n = c->gen_count;
    int rc = dedup_reserve(c, n);
    if (rc) return rc;
    ++c->dd_epoch;
    CK(c->dd_kept.ensure((size_t)n));
    launch_dedup_insert(dedup_view(c), c->gen_valid.as<unsigned char>(), c->gen_hash.as<unsigned long long>(), n,
                        c->dd_epoch, c->st);
    launch_dedup_mark(dedup_view(c), c->gen_valid.as<unsigned char>(), c->gen_hash.as<unsigned long long>(), n,
                      c->dd_epoch, c->dd_kept.as<unsigned char>(), c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_kept, c->dd_kept.p, (size_t)n, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (out_count) {
        int64_t k = 0;
        for (int64_t x = 0; x < n; ++x) k += out_kept[x] != 0;
        *out_count = k;
    }
    return L0S_OK;
}

int l0s_set_gram_mode(l0s_ctx* c, int mode) {
    if (!c) return fail(L0S_EINVAL, "null context");
    if (mode < L0S_GRAM_AUTO || mode > L0S_GRAM_OZAKI) return fail(L0S_EINVAL, "bad gram mode %d", mode);
    c->gram_mode = mode;
    return L0S_OK;
}

int l0s_stage_timings(l0s_ctx* c, double* out_ms) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    for (int x = 0; x < 4; ++x) out_ms[x] = 0.0;
    if (!c->stage_timed) return L0S_OK;
    out_ms[0] = elapsed(c->sev[0], c->sev[1]);
    out_ms[1] = c->stage_fused ? 0.0 : elapsed(c->sev[1], c->sev[2]);  // fused: one pass, out_ms[0]
    out_ms[2] = c->ms_gram_k;
    out_ms[3] = elapsed(c->sev[3], c->sev[4]);
    return L0S_OK;
}

int l0s_stage_loose_rows(l0s_ctx* c, int* out_count) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    *out_count = c->fix_count;
    return L0S_OK;
}

int l0s_stage_info(l0s_ctx* c, double* eta_out, int* ozaki_out) {
    if (!c || !c->staged) return fail(L0S_ESTATE, "l0s_stage must be called first");
    for (int t = 0; t < c->T; ++t) eta_out[t] = c->eta_h[(size_t)t];
    *ozaki_out = c->gram_ozaki ? 1 : 0;
    return L0S_OK;
}
