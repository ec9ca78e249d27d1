// fit3.cu -- screened exhaustive fit of every 3-tuple (i < j < k), fp64.
//
// Replaces the reference's per-tuple Householder sweep (score_tuples,
// lsq.py:113-156, driven by search._scan_range, search.py:174-199) with a
// lower bound computed from the staged normalized Gram:
//
//   per task t, column order [j, k, i] of the centered, unit-norm features,
//   LDL^T of the 3x3 correlation block plus the property row:
//     hoisted once per (j, k) pair:   d1 = 1 - C_jk^2,  s1 = (c_k - C_jk c_j) / d1,
//                                     base = |y_c|^2 - c_j^2 - (c_k - C_jk c_j)^2 / d1
//     per i (6 FP64 ops + 1 MUFU):    g1 = C_ik - C_jk C_ij,  e1 = g1 / d1,
//                                     d  = 1 - C_ij^2 - g1 e1,
//                                     w  = c_i - C_ij c_j - g1 s1,
//                                     ssr_t = base - w^2 / d
//   with the rigorous bound of fitcommon.cuh so that
//       lb = sum_t (ssr_t - A_t - B_t / d_t)  <=  the reference's pooled SSR.
//   lb is compared against the running threshold; the rare tuples that pass
//   are evaluated after the i-tile by the out-of-line slow path (exact bound,
//   conditioning, rank-rule certificate) and inserted into the warp's top-K'
//   list, or routed to the bit-exact kernel.
//
// Layout: one unit = 32 j (lanes) x KSPAN k (8 warps x P) x up to 128 i.
// The i-dependent Gram rows C[i, j-block], C[i, k-span], c_i are staged in
// shared memory by TMA (cp.async.bulk.tensor, mbarrier completion, double-buffered
// over IB-row tiles); the (j, k) state lives in registers.  Persistent CTAs pull
// units from an atomic counter.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "fitcommon.cuh"

namespace l0s {

using namespace fit;

namespace {

// (P, IB, MINB, UNROLL, NW) for 3-4 tasks; overridable (-DL0S_C34_P=... etc.) for tuning builds
#ifndef L0S_C34_P
#define L0S_C34_P 4
#endif
#ifndef L0S_C34_IB
#define L0S_C34_IB 24
#endif
#ifndef L0S_C34_MINB
#define L0S_C34_MINB 2
#endif
#ifndef L0S_C34_UNROLL
#define L0S_C34_UNROLL 1
#endif
#ifndef L0S_C34_NW
#define L0S_C34_NW 4
#endif
#ifndef L0S_C34_NBUF
#define L0S_C34_NBUF 2
#endif
#ifndef L0S_FIT_SLOT0
#define L0S_FIT_SLOT0 0
#endif
#ifndef L0S_PRUNE_ROWS
#define L0S_PRUNE_ROWS 4
#endif
#ifndef L0S_DIVFREE
#define L0S_DIVFREE 0
#endif
#ifndef L0S_WREL
#define L0S_WREL 0
#endif
// PA (phase A, NT > 1): before the per-group task loop, the first slot of every row of the tile is
// tested division-free, (K - theta) d - q < 0 with the same shrunk K (no MUFU, no per-group vote:
// one OR-reduction per tile); only groups with a survivor run the task loop.  A warp switches it
// off while more than PA_NUM / PA_DEN of its groups survive the first slot (dense near-ties: the
// test would only add work) and back on when fewer do.  Off: measured slower (C3 planted fit 1.565 ->
// 1.77 ms, random y 3.94 -> 4.00 ms; the per-group vote is not what limits the sweep, and the extra
// live ranges spill -- tools/tune_fit.py).
#ifndef L0S_PHASEA
#define L0S_PHASEA 0
#endif
#ifndef L0S_PA_NUM
#define L0S_PA_NUM 2
#endif
#ifndef L0S_PA_DEN
#define L0S_PA_DEN 5
#endif
// DF: the first task slot's test is division-free, (K - theta) d - q < 0, one FMA and no MUFU;
// only groups that survive it re-evaluate that slot with the reciprocal (as NT == 1 always does).
// WREL: tile buffers are released per warp (mbarrier + last-arriver refill), no CTA barrier per tile.
constexpr bool WREL = L0S_WREL;
// TSK: tile screen.  Before a unit's sweep every warp bounds its first task slot over each i-tile
// from row-block maxima of the Gram (k_tile_max): with a = max |C_ij|, b_p = max |C_ik_p|,
// c = max |c_i| over the tile's rows,
//   |g1| <= G1 = b_p + |C_jk| a,   d >= 1 - a^2 - G1^2 / d1,   |w| <= c + a |w0 - C_jk s1| + b_p |s1|,
// so when (K0 - theta) d_min > (w_max^2 + Bm) (1 + 4 kRcpRel) for every valid pair of the warp,
// every row of the tile would leave the first slot's test non-negative (pruned) and the warp
// skips the tile; tiles no warp needs are not loaded at all.  Results are unchanged: a skipped
// tuple's first-slot bound is at or above the threshold, which is the task pruning's own test.
#ifndef L0S_TSK_NOCALL
#define L0S_TSK_NOCALL 0
#endif
#ifndef L0S_TSKIP
#define L0S_TSKIP 1
#endif
constexpr bool TSK = L0S_TSKIP && !L0S_WREL;
constexpr int TSK_WORDS = 8;
// TSK_CTA: tiles no warp of the CTA needs are not loaded (else every tile is loaded and only the
// warps' compute is skipped)
#ifndef L0S_TSK_CTA
#define L0S_TSK_CTA 1
#endif
constexpr bool TSK_CTA = L0S_TSK_CTA;  // tile mask words per unit (units of more than 256 tiles are not screened)
struct CfgT {
    int P, IB, MINB, UNROLL, NW, NBUF;
};
// 3-4 tasks: two CTAs of 4 warps per SM, 4 pairs per thread, 24-row tiles (C3 fit 1.76 -> 1.55 ms
// against one CTA of 8 warps: a warp waiting at its CTA's tile barrier leaves the SM sub-partition
// to the other CTA's warp; 16 warps of 2 pairs spill at 128 registers, per-warp tile release,
// staging only the first task slot and 3-4 CTAs per SM were slower -- tools/tune_fit.py)
constexpr CfgT kCfg34{L0S_C34_P, L0S_C34_IB, L0S_C34_MINB, L0S_C34_UNROLL, L0S_C34_NW, L0S_C34_NBUF};
// (P, IB, MINB, UNROLL, NW) for 1, 2 and 5-8 tasks (-DL0S_C1_NW=... etc. for tuning builds).
// Measured on C3's features (tools/tune_fit.py): one task 4 CTAs x 4 warps (1.13 -> 1.04 ms
// against 2 x 8), two tasks 3 x 4 warps with 24-row tiles (1.31 -> 1.19 ms); 5-8 tasks keep
// one CTA of 8 warps (two CTAs of 4 were slower)
#ifndef L0S_C1_NW
#define L0S_C1_NW 4
#endif
#ifndef L0S_C1_MINB
#define L0S_C1_MINB 4
#endif
#ifndef L0S_C2_NW
#define L0S_C2_NW 4
#endif
#ifndef L0S_C2_MINB
#define L0S_C2_MINB 3
#endif
#ifndef L0S_C2_IB
#define L0S_C2_IB 24
#endif
#ifndef L0S_C58_P
#define L0S_C58_P 2
#endif
#ifndef L0S_C58_IB
#define L0S_C58_IB 16
#endif
#ifndef L0S_C58_MINB
#define L0S_C58_MINB 1
#endif
#ifndef L0S_C58_NW
#define L0S_C58_NW 8
#endif
constexpr CfgT kCfg1{4, 32, L0S_C1_MINB, 2, L0S_C1_NW, 2};
constexpr CfgT kCfg2{4, L0S_C2_IB, L0S_C2_MINB, 1, L0S_C2_NW, 2};
constexpr CfgT kCfg58{L0S_C58_P, L0S_C58_IB, L0S_C58_MINB, 1, L0S_C58_NW, 2};
// Per task count: P = (j,k) pairs per thread, IB = rows per i-tile, MINB = CTAs per SM,
// NW = warps per CTA (k-span = NW x P; the unit table follows it, fit3_kspan).
template <int NT>
struct Cfg {
    static constexpr CfgT c = (NT == 1) ? kCfg1 : (NT == 2 ? kCfg2 : (NT <= 4 ? kCfg34 : kCfg58));
    static constexpr int P = c.P;
    static constexpr int IB = c.IB;
    static_assert(IB >= 16, "fit3_tmax_doubles sizes the tile screen's tables for tile heights >= 16");
    static constexpr int NW = c.NW;
    static constexpr int NTH = NW * 32;
    static constexpr int KSPAN = NW * P;
    static constexpr int TS = IB * (32 + KSPAN + 2);  // C[i, j-block] | C[i, k-span] | (c_i, pad)
    // SLOT0: only the first task slot is staged (its rows feed every group); the other slots
    // are read from L2 by the few row groups that survive the first (task pruning)
    static constexpr bool SLOT0 = (NT > 1) && L0S_FIT_SLOT0;
    static constexpr int BS = SLOT0 ? TS : NT * TS;
    // tile ring depth (WREL: warps may run NBUF - 1 tiles apart; without it two buffers)
    static constexpr int NBUF = WREL ? c.NBUF : 2;
    static constexpr int MINB = c.MINB;
    static constexpr int UNROLL = c.UNROLL;  // rows of the i sweep in flight per thread
    // task pruning (NT > 1): rows per vote group, and per-thread smem slots for the
    // per-task constants (P x KS doubles: the total, then tasks 1..NT-1 for NT >= 3)
    static constexpr int R = (NT == 1) ? 1 : L0S_PRUNE_ROWS;
    static constexpr int KS = (NT >= 3) ? NT : 1;
    static constexpr size_t smem_bytes = (size_t)NBUF * BS * 8 + (size_t)NW * CAP * 16 + (size_t)NTH * P * KS * 8;
};

// Exact lower bound of one tuple (i < j < k) read straight from the Gram, with the
// arithmetic of the sweep (hoist on (j, k), i appended last).  Returns
// bit0 = bound trustworthy (conditioning, first-order validity, tightness),
// bit1 = the reference's rank rule certainly accepts the tuple; *lb in SSR units.
// Shared by the fit kernel's slow path and k_screen3 (so the tests exercise
// exactly the kernel's decision).  Kept out of line: the sweep's hot loop then
// carries only its (j, k) state in registers.
// *ub_out (optional) is the matching upper bound ssr_gram + A + B/d on the reference's SSR.
__device__ __noinline__ int eval_tuple3(const FitArgs& a, int64_t i, int64_t j, int64_t k, double* lb_out,
                                        double* ub_out = nullptr) {
    const int64_t m = a.m, mp = a.mp;
    double lb = 0.0, ub = 0.0;
    bool cond = true, rank_ok = true;
    for (int t = 0; t < a.T; ++t) {
        const double* Gt = a.G + (int64_t)t * mp * mp;
        const double Y2 = Gt[m * mp + m];
        const double w0 = Gt[m * mp + j];
        const double cjk = Gt[k * mp + j], ck = Gt[m * mp + k];
        const double d1 = fma(-cjk, cjk, 1.0);
        const double r1 = rcp_newton(d1);
        const double v1 = fma(-cjk, w0, ck);
        const double base = Y2 - w0 * w0 - v1 * v1 * r1;
        const double trh = 2.0 * r1;
        const double* rt_ = a.rho + (int64_t)t * m;
        const double rx = fmax(rt_[i], fmax(rt_[j], rt_[k]));
        double At, Bt, vk;
        task_bound(3, a.eta[t], ref_gamma(a.rowsd[t], 3, a.ref_fp32), rx, Y2, a.ynorm[t], trh, At, Bt, vk);
        if (!(d1 > 0.0) || !(vk * (1.0 + 3.0 * trh) <= FO_LIM)) cond = false;
        const double g0 = Gt[i * mp + j], ci = Gt[i * mp + m], gk = Gt[i * mp + k];
        const double D = fma(-g0, g0, 1.0);
        const double V = fma(-g0, w0, ci);
        const double g1 = fma(-cjk, g0, gk);
        const double e1 = g1 * r1;
        const double d = fma(-g1, e1, D);
        const double w = fma(-e1, v1, V);
        const double tr = trh + (1.0 + trh) / d;
        if (!(d > 0.0) || !(vk * (1.0 + 3.0 * tr) <= FO_LIM) || !(At + Bt / d <= (a.ref_fp32 ? LOOSE32 : LOOSE) * Y2)) cond = false;
        lb += base - At - fma(w, w, Bt) / d;
        ub += base + At - fma(w, w, -Bt) / d;
        const int64_t f[3] = {i, j, k};
        if (!rank_certain<3>(a, t, f, tr)) rank_ok = false;
    }
    *lb_out = lb;
    if (ub_out) *ub_out = ub;
    return (cond ? 1 : 0) | (rank_ok ? 2 : 0);
}

// The first task slot's hoisted state of a warp's P pairs, as the tile screen reads it.
template <int P>
struct PairSlot0 {
    double la[P];   // |C_jk|
    double sa[P];   // |s1| (1 + 2e-15)
    double wja[P];  // |c_j - C_jk s1| + 1e-15 (|C_jk| |s1| + |c_j|)
    double r1[P];   // 1 / (1 - C_jk^2), times (1 + 2e-14)
    double kq[P];   // the pair's first-slot margin (K0 - theta) * shrink (NT == 1: whole bound - theta),
                    // divided by (1 + 4 kRcpRel) (1 + 1e-12)
    double bm[P];   // an upper bound on max_t B_t
    unsigned cand;  // pairs a tile bound may retire: valid, not forced, kq > 0
    unsigned valid;
};

// Tile screen (TSK) of one warp over its unit's i-tiles.  Lane l gathers the row-block maxima
// (k_tile_max) of tile 32 w + l; groups of 4 tiles are tested first on the group's maxima, and
// only groups that fail are tested tile by tile.  Writes the warp's need bits (wneed[word]) and
// ORs them into the CTA's (need_cta[word]).  Out of line: its registers stay out of the sweep's.
template <int P, int IB>
__device__ __noinline__ void tile_screen(const FitArgs& a, const PairSlot0<P> ps, int lane, int kbase, int jb, int i_lo,
                                         int i_hi, int nib, unsigned* need_cta, unsigned* wneed) {
    const int64_t m = a.m;
    const bool all = __any_sync(L0S_FULL, (ps.valid & ~ps.cand) != 0u);
    const int nbk = (int)((m + IB - 1) / IB);
    const double* MT = a.tmax;                                   // [col][block], col <= m
    const double* MJ = a.tmax + (m + 1) * nbk + (int64_t)jb * nbk;  // this j-block's row
    // the bound of one row set with maxima (am, cm, ka[]): true = some pair still needs it.
    //   |g1| <= G1 = |C_jk| am + ka,  d >= 1 - am^2 - G1^2 / d1,  |w| <= cm + am |c_j - C_jk s1| + ka |s1|,
    // retired when K d_min > (w_max^2 + Bm); the sweep's own rounding (a few ulp of O(1) terms) and
    // its reciprocal's error are folded into the per-pair constants (PairSlot0) and the 1e-14 here
    auto needs = [&](double am, double cm, const double (&ka)[P]) {
        const double c1 = fma(-am, am, 1.0 - 1e-14);
        const double cw = cm * (1.0 + 1e-15);
        bool need = false;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (!((ps.valid >> p) & 1u)) continue;
            const double g1 = fma(ps.la[p], am, ka[p]);
            const double db = fma(-g1 * g1, ps.r1[p], c1);
            const double wb = fma(ka[p], ps.sa[p], fma(am, ps.wja[p], cw));
            const double q = fma(wb, wb, ps.bm[p]);
            // NaN / inf (flagged rows) fail the comparisons: needed
            need |= !(db > 1e-6 && fma(ps.kq[p], db, -q) > 0.0);
        }
        return __any_sync(L0S_FULL, need);
    };
    unsigned tests = 0;
    for (int wd = 0; wd * 32 < nib; ++wd) {
        unsigned word = all ? ~0u : 0u;
        if (!all) {
            double amx = 0.0, cmx = 0.0, kmx[P];
#pragma unroll
            for (int p = 0; p < P; ++p) kmx[p] = 0.0;
            const int tl = wd * 32 + lane;
            if (tl < nib) {
                const int r0 = i_lo + tl * IB, r1 = min(r0 + IB, i_hi);
                for (int b = r0 / IB; b <= (r1 - 1) / IB; ++b) {
                    amx = fmax(amx, MJ[b]);
                    cmx = fmax(cmx, MT[m * nbk + b]);
#pragma unroll
                    for (int p = 0; p < P; ++p) kmx[p] = fmax(kmx[p], MT[(kbase + p < m ? kbase + p : m - 1) * nbk + b]);
                }
            }
            // group maxima over lanes 4g .. 4g + 3 (tiles past nib hold zeros: harmless in a max)
            double gam = amx, gcm = cmx, gk[P];
#pragma unroll
            for (int p = 0; p < P; ++p) gk[p] = kmx[p];
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                gam = fmax(gam, __shfl_xor_sync(L0S_FULL, gam, o));
                gcm = fmax(gcm, __shfl_xor_sync(L0S_FULL, gcm, o));
#pragma unroll
                for (int p = 0; p < P; ++p) gk[p] = fmax(gk[p], __shfl_xor_sync(L0S_FULL, gk[p], o));
            }
            const int nt = min(32, nib - wd * 32);
            for (int g = 0; g * 4 < nt; ++g) {
                double ka[P];
#pragma unroll
                for (int p = 0; p < P; ++p) ka[p] = __shfl_sync(L0S_FULL, gk[p], 4 * g);
                ++tests;
                if (!needs(__shfl_sync(L0S_FULL, gam, 4 * g), __shfl_sync(L0S_FULL, gcm, 4 * g), ka)) continue;
                for (int bb = 4 * g; bb < min(4 * g + 4, nt); ++bb) {
#pragma unroll
                    for (int p = 0; p < P; ++p) ka[p] = __shfl_sync(L0S_FULL, kmx[p], bb);
                    ++tests;
                    if (needs(__shfl_sync(L0S_FULL, amx, bb), __shfl_sync(L0S_FULL, cmx, bb), ka)) word |= 1u << bb;
                }
            }
        }
        if (lane == 0) {
            wneed[wd] = word;
            atomicOr(&need_cta[wd], word);
        }
    }
    if (lane == 0 && tests && a.n_screen) atomicAdd(a.n_screen, (unsigned long long)tests);
}

// The sweep's static shared state (one instance per CTA, whichever instantiation runs).
template <int NT>
struct FitShared {
    using C = Cfg<NT>;
    int unit;
    int tord[NT];
    unsigned char force[C::NBUF][C::IB];  // iforce flags of the staged rows
    int fany[C::NBUF];                    // any of them set
    alignas(8) unsigned long long bar[C::NBUF];  // TMA completion, one per tile buffer
    alignas(8) unsigned long long hbar;          // TMA completion of the unit's hoist block
    unsigned rel[C::NBUF];                       // WREL: warps done with the buffer's tile
    double th;                                   // the unit's shared threshold
    unsigned need[TSK_WORDS];                    // TSK: tiles some warp needs
    unsigned wneed[C::NW][TSK_WORDS];            // TSK: tiles this warp needs
    double ts[4][NT];  // Y2, gamma, eta, A0 = 4 gamma |y_c| |y| (task_bound's constant term)
    // the unit's hoist inputs besides C[k, j] (TMA block), per task slot: c_j and max(rho_cap,
    // rho_j) over the j-block, c_k and rho_k over the k-span
    double hu[NT][4][32];
};

template <int NT, bool SCR>
__device__ __forceinline__ void fit3_sweep(const FitArgs& a, FitShared<NT>& S) {
    using C = Cfg<NT>;
    constexpr bool TSKB = TSK && SCR;  // this instantiation runs the tile screen
    constexpr int NW3 = C::NW, NT3 = C::NTH;
    constexpr int P = C::P, IB = C::IB, TS = C::TS, BS = C::BS, KSPAN = C::KSPAN, R = C::R, NB = C::NBUF;
    constexpr bool DF = L0S_DIVFREE && NT > 1 && !C::SLOT0 && (P % 2 == 0);
    constexpr bool PA = L0S_PHASEA && NT > 1 && !DF && !C::SLOT0 && (P % 2 == 0);
    constexpr int NG = IB / R;  // vote groups per tile
    static_assert(!PA || NG <= 32, "group bits in one word");
    int pa_tot = 0, pa_surv = 0;  // groups seen / surviving the first slot (warp-uniform, decayed)
    extern __shared__ __align__(128) double sm[];
    auto& s_unit = S.unit;
    auto& s_tord = S.tord;
    auto& s_force = S.force;
    auto& s_fany = S.fany;
    auto& s_bar = S.bar;
    auto& s_hbar = S.hbar;
    auto& s_rel = S.rel;
    auto& s_th = S.th;
    auto& s_need = S.need;
    auto& s_wneed = S.wneed;
    auto& s_ts = S.ts;
    auto& s_hu = S.hu;
    unsigned long long n_ev = 0;                            // row-group task evaluations (warp-uniform)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m = a.m, mp = a.mp;
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) {
            s_rel[b] = 0u;
            mbar_init(&s_bar[b], 1);
        }
        mbar_init(&s_hbar, 1);
        mbar_fence_init();
        // sweep order of the tasks: largest |y_c|^2 first, so that the first task's share of the
        // bound alone already exceeds the threshold for almost every row (task pruning below);
        // with more than NT tasks the slots take the NT largest (a subset bounds the pooled SSR)
        double y2[NT];
        int cnt = 0;
        for (int t = 0; t < a.T; ++t) {
            const double v = a.G[(int64_t)t * mp * mp + m * mp + m];
            int z;
            if (cnt < NT) {
                z = cnt++;
            } else if (v > y2[NT - 1]) {
                z = NT - 1;
            } else {
                continue;
            }
            y2[z] = v;
            s_tord[z] = t;
            for (; z > 0 && y2[z] > y2[z - 1]; --z) {
                const double w = y2[z];
                y2[z] = y2[z - 1];
                y2[z - 1] = w;
                const int q = s_tord[z];
                s_tord[z] = s_tord[z - 1];
                s_tord[z - 1] = q;
            }
        }
    }
    __syncthreads();
    // unit-independent per-task scalars of the hoist, in slot order, once per CTA (shared
    // memory instead of a global load chain per unit)
    if (tid < NT) {
        const int tk = s_tord[tid];
        const double Y2 = a.G[(int64_t)tk * mp * mp + m * mp + m], gam = ref_gamma(a.rowsd[tk], 3, a.ref_fp32);
        s_ts[0][tid] = Y2;
        s_ts[1][tid] = gam;
        s_ts[2][tid] = a.eta[tk];
        s_ts[3][tid] = 4.0 * gam * sqrt(Y2) * a.ynorm[tk];
    }
    // the unit's hoist inputs besides C[k, j] (TMA block below), per task slot, staged by all
    // threads with coalesced loads: c_j and max(rho_cap, rho_j) over the j-block, c_k and rho_k
    // over the k-span (a per-pair global load chain stalled the hoist on the LSU queue)
    static_assert(KSPAN <= 32, "k-span staged in 32-wide rows");
    __syncthreads();
    const int* tord = s_tord;  // read where the hoist / tile loads need it (rare)
    unsigned parity = 0u, hpar = 0u;  // full-barrier phase bit per tile buffer
    // TSKB: the block maxima must be those of this kernel's first slot (k_tile_max picks the same task)
    const bool tsk_on = TSKB && a.tmax != nullptr &&
                        a.tmax[(m + 1 + (m + 31) / 32) * ((m + IB - 1) / IB)] == (double)tord[0];
    // The unit's hoist block goes through TMA into tile buffers 1.. (idle until the sweep's first
    // prefetch): per task slot C[k-span, j-block] (KSPAN x 32).
    constexpr int HS = KSPAN * 32;  // doubles per task slot: C[k-span, j-block]
#ifndef L0S_HOIST_TMA
#define L0S_HOIST_TMA 1
#endif
    constexpr bool HT = L0S_HOIST_TMA && NT * HS <= (NB - 1) * BS;  // else the hoist reads L2
    // per-thread constants, touched by the hoist, threshold updates and pruned rows:
    // sK[0][p] = sum_t (base_t - A_t) (NT >= 3: sK[t][p] = (base_t - A_t) * shrink, t >= 1)
    // (slot-major, thread-minor: conflict-free per-thread accesses)
    double* sKb = sm + NB * BS + 2 * NW3 * CAP + tid;
    auto sK = [&](int idx) -> double& { return sKb[idx * NT3]; };
    const double shrink = (NT == 1) ? 1.0 : (1.0 - 2.0 * kRcpRel);
    WarpCands wc{sm + NB * BS + warp * CAP, reinterpret_cast<int64_t*>(sm + NB * BS + NW3 * CAP) + warp * CAP, 0,
                 a.collect == 1 ? a.theta0 : ord_dec(*(volatile unsigned long long*)a.theta_g), 0};
    const int64_t* B2 = a.binom + 2 * (m + 1);
    const int64_t* B3 = a.binom + 3 * (m + 1);

    // tiles per task (slot t holds task tord[t]), staged by TMA (one elected thread,
    // completion on s_bar[buf]): C[i, j-block] (IB x 32), C[i, k-span] (IB x KSPAN), (c_i, pad) (IB x 2)
    // Issued by one whole warp (`by`): its lanes write the rows' iforce flags, its lane 0 the TMA.
    auto load_tiles = [&](int buf, int ib0, int j0, int k0, int by = 0) {
        if (warp == by) {  // the rows' iforce flags and whether any is set
            unsigned any = 0u;
#pragma unroll
            for (int r0 = 0; r0 < IB; r0 += 32) {
                const int r = r0 + lane;
                const unsigned char fl = (r < IB && ib0 + r < m) ? a.iforce[ib0 + r] : 0;
                if (r < IB) s_force[buf][r] = fl;
                any |= __ballot_sync(L0S_FULL, fl != 0);
            }
            if (lane == 0) s_fany[buf] = any != 0u;
            __syncwarp();  // the flags precede lane 0's arrive (release) on the tile's barrier
        }
        if (warp == by && lane == 0) {
            double* base = sm + buf * BS;
            fence_proxy_async();
            mbar_expect_tx(&s_bar[buf], (unsigned)(BS * sizeof(double)));
#pragma unroll
            for (int t = 0; t < (C::SLOT0 ? 1 : NT); ++t) {
                const int row = (int)(tord[t] * mp) + ib0;
                double* Tt = base + t * TS;
                tma_load_2d(Tt, &a.tmJ, j0, row, &s_bar[buf]);
                tma_load_2d(Tt + IB * 32, &a.tmK, k0, row, &s_bar[buf]);
                // TMA box starts must be 16-byte aligned: the pair of columns (m & ~1, +1) holds c_i
                tma_load_2d(Tt + IB * (32 + KSPAN), &a.tmC, (int)(m & ~(int64_t)1), row, &s_bar[buf]);
            }
        }
    };
    auto wait_tiles = [&](int buf) {
        mbar_wait(&s_bar[buf], (parity >> buf) & 1u);
        parity ^= 1u << buf;
    };

    for (;;) {
        if (tid == 0) s_unit = atomicAdd(a.unit_counter, 1);
        __syncthreads();
        const int u = s_unit;
        __syncthreads();
        if (u >= a.n_units) break;
        const int4 U = a.units[u];
        const int j0 = U.x * 32, k0 = U.y * KSPAN;
        const int j = j0 + lane;
        const int kbase = k0 + warp * P;
        const int i_lo = U.z, i_hi = U.w;
        if (TSKB && tid < TSK_WORDS) s_need[tid] = 0u;  // ordered before the screen's atomics by the hoist's barriers
        double* Hb = sm + BS;  // tile buffers 1..
        if (HT && tid == 0) {
            fence_proxy_async();  // the previous unit's reads of buffer 1 precede these writes
            mbar_expect_tx(&s_hbar, (unsigned)(NT * HS * sizeof(double)));
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                tma_load_2d(Hb + t * HS, &a.tmH, j0, (int)(tord[t] * mp) + k0, &s_hbar);
            }
        }
        if (!TSKB) load_tiles(0, i_lo, j0, k0);  // (with the screen: the first needed tile, below)
        for (int x = tid; x < NT * 128; x += NT3) {
            const int t = x >> 7, w = (x >> 5) & 3, l = x & 31;
            const int tk = tord[t];
            const int f = (w < 2 ? j0 : k0) + l, ff = f < m ? f : (int)m - 1;
            double v;
            if (w == 0 || w == 2)
                v = a.G[(int64_t)tk * mp * mp + m * mp + f];  // c_j / c_k (columns < mp: padded, finite)
            else
                v = w == 1 ? fmax(a.rho_cap[tk], a.rho[(int64_t)tk * m + ff]) : a.rho[(int64_t)tk * m + ff];
            s_hu[t][w][l] = v;
        }
        if (a.collect != 1 && warp == NW3 - 1) {
            // shared threshold: the global bound histogram and the other warps' lists (one warp
            // per CTA reads them; the histogram scan is a long load chain)
            const double th = fmin(hist_theta(a, lane), ord_dec(*(volatile unsigned long long*)a.theta_g));
            if (lane == 0) {
                s_th = th;
                atomicMin(a.theta_g, ord_enc(th));
            }
        }
        __syncthreads();
        if (a.collect != 1 && s_th < wc.theta) wc.theta = s_th;

        if (HT) {
            mbar_wait(&s_hbar, hpar);
            hpar ^= 1u;
        }
        // ---------------- tile screen (TSKB, out of line: its registers stay out of the sweep's) ----------------
        // Before the hoist, from the first slot's exact hoist of each pair plus, over every slot, the
        // finiteness / conditioning flags and an upper bound on Bm = max_t B_t (1/d1 rounded up in
        // float): a unit no warp needs a tile of skips the hoist and the sweep altogether.
        const int nib = (i_hi - i_lo + IB - 1) / IB;
        const bool scr = tsk_on && nib <= 32 * TSK_WORDS;
        if constexpr (TSKB) {
            if (scr && !L0S_TSK_NOCALL) {
                PairSlot0<P> ps;
                const double wj0 = s_hu[0][0][lane];
                ps.valid = 0u;
                ps.cand = 0u;
                // slots 1..: B_t = 3 K_t Y2_t (1 + 2/d1_t) <= 6 (eta + gamma rho) Y2 (1 + 2/d1) with
                // each factor's maximum over the slots (rho over the pair's j and k)
                double etx = 0.0, gmx = 0.0, y2x = 0.0, rjx = 0.0;
                bool fj = true;
#pragma unroll
                for (int t = 1; t < NT; ++t) {
                    y2x = fmax(y2x, s_ts[0][t]);
                    gmx = fmax(gmx, s_ts[1][t]);
                    etx = fmax(etx, s_ts[2][t]);
                    rjx = fmax(rjx, s_hu[t][1][lane]);
                    fj = fj && isfinite(s_hu[t][0][lane]);
                }
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int k = kbase + p;
                    bool ok = fj, fin = fj;
                    double bm;
                    {
                        const double Y2 = s_ts[0][0];
                        const double cjk = HT ? Hb[(k - k0) * 32 + lane] : a.G[(int64_t)tord[0] * mp * mp + (int64_t)k * mp + j];
                        const double ck = s_hu[0][2][k - k0];
                        const double d1 = fma(-cjk, cjk, 1.0);
                        const double r1 = rcp_newton(d1);
                        const double v1 = fma(-cjk, wj0, ck);
                        const double base = Y2 - wj0 * wj0 - v1 * v1 * r1;
                        const double trh = 2.0 * r1;
                        double At, Bt, vk;
                        const double rh = fmax(s_hu[0][1][lane], s_hu[0][3][k - k0]);
                        task_bound_a0(3, s_ts[2][0], s_ts[1][0], rh, Y2, s_ts[3][0], trh, At, Bt, vk);
                        if (!(d1 > 0.0) || !(vk * (1.0 + 3.0 * trh) <= FO_LIM)) ok = false;
                        if (!isfinite(cjk + ck + wj0)) fin = false;
                        bm = Bt;
                        const double s1v = v1 * r1, la = fabs(cjk), sa = fabs(s1v);
                        // the sweep's rounding folded in (PairSlot0; a few ulp of O(1) terms)
                        ps.la[p] = la;
                        ps.sa[p] = sa * (1.0 + 2e-15);
                        ps.wja[p] = fabs(fma(-cjk, s1v, wj0)) + 1e-15 * fma(la, sa, fabs(wj0));
                        ps.r1[p] = r1 * (1.0 + 2e-14);
                        const double kq = (NT == 1) ? (base - At) - wc.theta : ((base - At) - wc.theta) * shrink;
                        ps.kq[p] = kq * (1.0 / ((1.0 + 4.0 * kRcpRel) * (1.0 + 1e-12)));
                    }
                    if (NT > 1) {
                        double dmin = 1.0, rkx = 0.0;
#pragma unroll
                        for (int t = 1; t < NT; ++t) {
                            const double cjk = HT ? Hb[t * HS + (k - k0) * 32 + lane] : a.G[(int64_t)tord[t] * mp * mp + (int64_t)k * mp + j];
                            dmin = fmin(dmin, fma(-cjk, cjk, 1.0));
                            rkx = fmax(rkx, s_hu[t][3][k - k0]);
                            if (!isfinite(cjk + s_hu[t][2][k - k0])) fin = false;
                        }
                        // 1/d1 from above: d1 rounded down to float, its reciprocal rounded up (0 or
                        // denormal: inf, the pair is then never retired)
                        const double rup = (double)__frcp_ru(__double2float_rd(dmin));
                        const double kx = 2.0 * fma(gmx, fmax(rjx, rkx), etx) * (1.0 + 1e-12);
                        bm = fmax(bm, 3.0 * kx * y2x * (1.0 + 2.0 * rup) * (1.0 + 1e-12));
                        if (!(dmin > 0.0)) ok = false;
                    }
                    ps.bm[p] = fmax(bm, 1e-300);
                    if (j < k && k < m && fin) ps.valid |= 1u << p;
                    if (ok && fin && ps.kq[p] > 0.0 && bm == bm) ps.cand |= 1u << p;
                }
                tile_screen<P, IB>(a, ps, lane, kbase, U.x, i_lo, i_hi, nib, s_need, s_wneed[warp]);
            } else if (lane < TSK_WORDS) {  // no screen: every tile (the sweep reads the masks alone)
                s_wneed[warp][lane] = ~0u;
                atomicOr(&s_need[lane], ~0u);
            }
            __syncthreads();
            unsigned anyw = 0u;
#pragma unroll
            for (int w = 0; w < TSK_WORDS; ++w) anyw |= s_need[w];
            if (anyw == 0u) continue;  // no warp needs a tile of this unit: no hoist, no sweep
        }

        // ---------------- hoist: (j, k_p) state per task (slot order) ----------------
        // L10 = C_jk, rd1 = 1/(1 - C_jk^2), s1 = rd1 (c_k - C_jk c_j); the bound's B_t/d term
        // uses Bm = max_t B_t per pair, so the sweep needs one extra register per pair only
        double L10[P][NT], rd1[P][NT], s1[P][NT], w0[NT], Kq[P], Bm[P];
        double K1r[P];  // NT == 2: task slot 1's (base - A) * shrink in registers
        unsigned valid = 0, bad = 0, forced = 0;
#pragma unroll
        for (int t = 0; t < NT; ++t) w0[t] = s_hu[t][0][lane];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int k = kbase + p;
            double kr = 0.0, bm = 0.0;
            bool isbad = false, isnan_ = false;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double Y2 = s_ts[0][t];
                const double cjk = HT ? Hb[t * HS + (k - k0) * 32 + lane]
                                      : a.G[(int64_t)tord[t] * mp * mp + (int64_t)k * mp + j];
                const double ck = s_hu[t][2][k - k0];
                const double d1 = fma(-cjk, cjk, 1.0);
                const double r1 = rcp_newton(d1);
                const double v1 = fma(-cjk, w0[t], ck);
                const double base = Y2 - w0[t] * w0[t] - v1 * v1 * r1;
                const double trh = 2.0 * r1;
                double At, Bt, vk;
                // rho of the hoisted pair (the sweep feature's rho is covered by rho_cap or s_force)
                const double rh = fmax(s_hu[t][1][lane], s_hu[t][3][k - k0]);
                task_bound_a0(3, s_ts[2][t], s_ts[1][t], rh, Y2, s_ts[3][t], trh, At, Bt, vk);
                L10[p][t] = cjk;
                rd1[p][t] = r1;
                s1[p][t] = v1 * r1;
                kr += base - At;
                if (t == 0) Kq[p] = base - At;  // slot 0's share (the sweep's first partial bound)
                if constexpr (NT == 2) {
                    if (t == 1) K1r[p] = (base - At) * shrink;
                } else if constexpr (NT >= 3) {
                    if (t >= 1) sK(t * P + p) = (base - At) * shrink;
                }
                bm = fmax(bm, Bt);
                if (!(d1 > 0.0) || !(vk * (1.0 + 3.0 * trh) <= FO_LIM)) isbad = true;
                if (cjk != cjk || ck != ck || w0[t] != w0[t]) isnan_ = true;
            }
            sK(p) = kr;
            Bm[p] = fmax(bm, 1e-300);  // q = w^2 + Bm > 0: d <= 0 always reads as "below theta"
            if (j < k && k < m && !isnan_) valid |= 1u << p;
            if (isbad) bad |= 1u << p;
        }
        // Kq = (first slot's share - theta) * shrink for NT > 1 (the remaining slots are added as the
        // rows survive; DF: unshrunk, the first slot's test is division-free), (total - theta) for
        // NT == 1; forced = pairs whose whole bound is below theta
        double K0[P];
#pragma unroll
        for (int p = 0; p < P; ++p) K0[p] = Kq[p];
        auto set_kq = [&]() {
            forced = bad;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double x = sK(p) - wc.theta;
                if (!(x > 0.0)) forced |= 1u << p;
                Kq[p] = (NT == 1) ? x : (DF ? (K0[p] - wc.theta) : (K0[p] - wc.theta) * shrink);
            }
        };
        set_kq();
        __syncthreads();  // every warp is done with the hoist block: buffer 1 may take tile 1

        // first tile at or after b that some warp needs (TSKB; the masks are all ones without a screen)
        // (word-wise, and made warp-uniform by a reduction so that the sweep's addressing stays scalar)
        auto next_needed = [&](int b) -> int {
            if constexpr (TSKB && TSK_CTA) {
                int r = b;  // past the screened range: every tile
                if (b < 32 * TSK_WORDS) {
                    r = nib;
                    for (int w = b >> 5; w < TSK_WORDS && w * 32 < nib; ++w) {
                        unsigned msk = s_need[w];
                        if (w == (b >> 5)) msk &= ~0u << (b & 31);
                        if (msk) {
                            r = w * 32 + __ffs(msk) - 1;
                            break;
                        }
                    }
                }
                return (int)__reduce_min_sync(L0S_FULL, (unsigned)min(r, nib));
            } else {
                return b;
            }
        };

        // ---------------- sweep i ----------------
        if (WREL)
            for (int b = 1; b < NB && b < nib; ++b) load_tiles(b, i_lo + b * IB, j0, k0);
        // the screened sweep stages the first needed tile only now (buffer 0; the hoist used 1..)
        if (TSKB) {
            const int bf = next_needed(0);
            if (bf < nib) load_tiles(0, i_lo + bf * IB, j0, k0);
        }
        // needed tiles in order, alternating between the two buffers (pb); the next one is staged
        // while this one is swept
        int pb = 0;
        for (int bi = next_needed(0); bi < nib; bi = next_needed(bi + 1), pb ^= 1) {
            const int buf = WREL ? bi % NB : (TSKB ? pb : (bi & 1));
            const int ib0 = i_lo + bi * IB;
            if (!WREL) {
                const int bn = next_needed(bi + 1);
                if (bn < nib) load_tiles(buf ^ 1, i_lo + bn * IB, j0, k0);
            }
            wait_tiles(buf);
#ifndef L0S_TILE_BAR0
#define L0S_TILE_BAR0 1
#endif
            // s_force of this tile would not need a CTA barrier (its writers' __syncwarp precedes
            // the releasing arrive on the tile's mbarrier, which every reader acquires), but the
            // warps kept in step run faster (C3 fit 1.557 ms with it, 1.571 without; random y
            // 3.93 / 4.09 ms -- tools/tune_fit.py)
            if (L0S_TILE_BAR0 && !WREL) __syncthreads();
            const double* T0 = sm + buf * BS;
            // a clean tile (warp-uniform): every row is below every lane's j and inside the unit,
            // and no row is iforce-flagged -- a row's pending bits are then just the sign bits
            const bool clean = ib0 + IB <= i_hi && ib0 + IB <= j0 && !s_fany[buf];
            // pending slow-path tuples of this tile: bit (ii * P + p)
            constexpr int NPW = (IB * P + 31) / 32;  // pending-bit words
            constexpr int IPW = 32 / P;              // rows per word
            static_assert(IPW % R == 0, "vote groups must not straddle pending words");
            unsigned pend[NPW];
            // one task slot of one row: acc[p] -= (w^2 + Bm) / d  (NT == 1: acc = acc d - q)
            // lb_t = base_t - A_t - (w^2 + B_t)/d >= base_t - A_t - (w^2 + Bm)/d
            auto task_row = [&](double (&acc)[P], int t, int ii) {
                double g0, ci, gk[P];
                if (C::SLOT0 && t > 0) {
                    // surviving group: this slot's row straight from L2 (rows < mp: padded rows are finite)
                    const double* Gi = a.G + (int64_t)tord[t] * mp * mp + (int64_t)(ib0 + ii) * mp;
                    g0 = Gi[j];
                    ci = Gi[m];
#pragma unroll
                    for (int p = 0; p < P; p += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(Gi + kbase + p);
                        gk[p] = v.x;
                        gk[p + 1] = v.y;
                    }
                } else {
                const double* Tt = T0 + (C::SLOT0 ? 0 : t) * TS;
                g0 = Tt[ii * 32 + lane];
                ci = Tt[IB * (32 + KSPAN) + 2 * ii + (int)(m & 1)];
                if constexpr (P == 1) {
                    gk[0] = Tt[IB * 32 + ii * KSPAN + warp];
                } else {
#pragma unroll
                    for (int p = 0; p < P; p += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(Tt + IB * 32 + ii * KSPAN + warp * P + p);
                        gk[p] = v.x;
                        gk[p + 1] = v.y;
                    }
                }
                }
                const double D = fma(-g0, g0, 1.0);
                const double V = fma(-g0, w0[t], ci);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double g1 = fma(-L10[p][t], g0, gk[p]);
                    const double e1 = g1 * rd1[p][t];
                    const double w = fma(-g1, s1[p][t], V);
                    const double d = fma(-g1, e1, D);
                    const double q = fma(w, w, Bm[p]);
                    if (NT == 1)
                        acc[p] = fma(acc[p], d, -q);  // (K - theta) d - q; d <= 0 also passes
                    else
                        acc[p] = fma(-q, fabs(rcp_sweep(d)), acc[p]);  // 1/|d|: d <= 0 drives acc down
                }
            };
            // DF: slot 0 of one row, division-free: sign bit of (K0 - theta) d - q for every pair
            // (d <= 0 with K0 > theta: negative since q > 0 -- still alive, as in the NT == 1 form)
            auto task_row_df = [&](unsigned& sg, int ii) {
                const double* Tt = T0;
                const double g0 = Tt[ii * 32 + lane];
                const double ci = Tt[IB * (32 + KSPAN) + 2 * ii + (int)(m & 1)];
                double gk[P];
#pragma unroll
                for (int p = 0; p < P; p += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(Tt + IB * 32 + ii * KSPAN + warp * P + p);
                    gk[p] = v.x;
                    gk[p + 1] = v.y;
                }
                const double D = fma(-g0, g0, 1.0);
                const double V = fma(-g0, w0[0], ci);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double g1 = fma(-L10[p][0], g0, gk[p]);
                    const double e1 = g1 * rd1[p][0];
                    const double w = fma(-g1, s1[p][0], V);
                    const double d = fma(-g1, e1, D);
                    const double q = fma(w, w, Bm[p]);
                    sg |= (unsigned)__double2hiint(fma(Kq[p], d, -q));
                }
            };
            // PA: slot 0 of one row, division-free with the shrunk Kq: sign bit of Kq d - q (alive when
            // negative: d > 0 and lb_0 below theta, or d <= 0), OR-ed into sg
            auto task_row_a = [&](unsigned& sg, int ii) {
                const double* Tt = T0;
                const double g0 = Tt[ii * 32 + lane];
                const double ci = Tt[IB * (32 + KSPAN) + 2 * ii + (int)(m & 1)];
                double gk[P];
#pragma unroll
                for (int p = 0; p < P; p += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(Tt + IB * 32 + ii * KSPAN + warp * P + p);
                    gk[p] = v.x;
                    gk[p + 1] = v.y;
                }
                const double D = fma(-g0, g0, 1.0);
                const double V = fma(-g0, w0[0], ci);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double g1 = fma(-L10[p][0], g0, gk[p]);
                    const double e1 = g1 * rd1[p][0];
                    const double w = fma(-g1, s1[p][0], V);
                    const double d = fma(-g1, e1, D);
                    const double q = fma(w, w, Bm[p]);
                    sg |= (unsigned)__double2hiint(fma(Kq[p], d, -q));
                }
            };
            // phase A (PA): division-free first-slot test of every row, one bit per group
            unsigned gal = ~0u;
            bool use_a = false;
            if constexpr (PA) {
                use_a = pa_surv * L0S_PA_DEN <= pa_tot * L0S_PA_NUM;
                if (use_a) {
                    unsigned lb = 0u;
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        unsigned sg = 0u;
#pragma unroll
                        for (int r = 0; r < R; ++r) task_row_a(sg, g * R + r);
                        lb |= (sg >> 31) << g;
                    }
                    gal = __reduce_or_sync(L0S_FULL, lb);
                    n_ev += NG;
                    pa_tot += NG;
                    pa_surv += __popc(gal);
                } else {
                    pa_tot += NG;  // pa_surv counts the groups passing the first slot's vote below
                }
                if (pa_tot >= 512) {
                    pa_tot >>= 1;
                    pa_surv >>= 1;
                }
            }
            // TSKB: a warp whose pairs all clear this tile's bound has nothing pending in it
            const bool wneed = !TSKB || __any_sync(L0S_FULL, bi >= 32 * TSK_WORDS || ((s_wneed[warp][bi >> 5] >> (bi & 31)) & 1u));
#pragma unroll
            for (int pw = 0; pw < NPW; ++pw) pend[pw] = 0u;
            if (wneed) {
#pragma unroll
            for (int pw = 0; pw < NPW; ++pw) {
                unsigned word = 0u;
#pragma unroll(C::UNROLL)
                for (int ig = 0; ig < IPW; ig += R) {
                    double acc[R][P];
                    // Task pruning: every task's reference SSR is >= 0, so the slots swept so far
                    // already bound the pooled SSR from below.  Once no (row, lane, pair) of the
                    // group is below theta on them, the group is done (warp-uniform exit).
                    bool live = true;
                    if constexpr (DF) {
                        unsigned sg = 0u;
#pragma unroll
                        for (int r = 0; r < R; ++r) task_row_df(sg, pw * IPW + ig + r);
                        ++n_ev;
                        live = __any_sync(L0S_FULL, (int)sg < 0);
                        if (live) {  // survivors: slot 0 again with the reciprocal, then the others
#pragma unroll
                            for (int r = 0; r < R; ++r) {
#pragma unroll
                                for (int p = 0; p < P; ++p) acc[r][p] = Kq[p] * shrink;
                                task_row(acc[r], 0, pw * IPW + ig + r);
                            }
                            ++n_ev;
                        }
                    } else if (PA && !((gal >> ((pw * IPW + ig) / R)) & 1u)) {
                        live = false;  // no lane's first slot is below theta (phase A)
                    } else {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
#pragma unroll
                            for (int p = 0; p < P; ++p) acc[r][p] = Kq[p];
                            task_row(acc[r], 0, pw * IPW + ig + r);
                        }
                        ++n_ev;
                    }
#pragma unroll
                    for (int t = 1; t < NT && live; ++t) {
                        // sign bits OR-ed as integers (acc < 0 or -0: still alive; cheaper than
                        // predicate chains, which the compiler turns into an fmin reduction)
                        unsigned sgn = 0u;
#pragma unroll
                        for (int r = 0; r < R; ++r)
#pragma unroll
                            for (int p = 0; p < P; ++p) sgn |= (unsigned)__double2hiint(acc[r][p]);
                        if (!__any_sync(L0S_FULL, (int)sgn < 0)) {
                            live = false;
                            break;
                        }
                        if (PA && t == 1 && !use_a) ++pa_surv;
                        double kt[P];
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            if constexpr (NT == 2)
                                kt[p] = K1r[p];
                            else
                                kt[p] = sK(t * P + p);
                        }
#pragma unroll
                        for (int r = 0; r < R; ++r) {
#pragma unroll
                            for (int p = 0; p < P; ++p) acc[r][p] += kt[p];
                            task_row(acc[r], t, pw * IPW + ig + r);
                        }
                        ++n_ev;
                    }
                    if (clean) {
                        unsigned bits = 0u;  // sign bits of the group, row-major (r * P + p)
                        if (live) {
#pragma unroll
                            for (int r = 0; r < R; ++r)
#pragma unroll
                                for (int p = 0; p < P; ++p)
                                    bits |= ((unsigned)__double2hiint(acc[r][p]) >> 31) << (r * P + p);
                        }
                        unsigned fv = forced, vv = valid;  // replicate the per-pair masks over the R rows
#pragma unroll
                        for (int r = 1; r < R; ++r) {
                            fv |= forced << (r * P);
                            vv |= valid << (r * P);
                        }
                        word |= ((bits | fv) & vv) << (ig * P);
                    } else {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const int ii = pw * IPW + ig + r;
                            const int i = ib0 + ii;
                            unsigned pass = forced;
                            if (live) {
#pragma unroll
                                for (int p = 0; p < P; ++p) pass |= ((unsigned)__double2hiint(acc[r][p]) >> 31) << p;
                            }
                            if (s_force[buf][ii]) pass |= (1u << P) - 1;  // rho_i above rho_cap: needs the actual rho
                            pass &= valid;
                            if (!(i < j && i < i_hi)) pass = 0;
                            word |= pass << ((ig + r) * P);
                        }
                    }
                }
                pend[pw] = word;
            }
            }

            // ---------------- slow path (rare), after the tile ----------------
            drain_pending<NPW>(
                a, pend, wc, lane,
                [&](int b, double* lbv, int64_t* rkv) -> int {
                    const int ii = b / P, p = b % P;
                    const int i = ib0 + ii, k = kbase + p;
                    *rkv = a.N_total - 1 - (B3[m - 1 - i] + B2[m - 1 - j] + (m - 1 - k));
                    if (a.ranged && (*rkv < a.rank_lo || *rkv >= a.rank_hi)) return 0;
                    if ((bad >> p) & 1u) return 2;
                    return eval_tuple3(a, i, j, k, lbv) == 3 ? 1 : 2;
                },
                set_kq);
            if (WREL) {
                // per-warp release instead of a CTA barrier: the last warp done with this buffer
                // refills it with tile bi + 2 (a warp deep in its slow path delays only that load)
                __syncwarp();
                unsigned last = 0;
                if (lane == 0) last = atomicAdd(&s_rel[buf], 1u) == NW3 - 1;
                last = __shfl_sync(L0S_FULL, last, 0);
                if (last) {
                    if (lane == 0) s_rel[buf] = 0u;
                    if (bi + NB < nib) load_tiles(buf, ib0 + NB * IB, j0, k0, warp);
                }
            } else {
                __syncthreads();
            }
        }
        if (WREL) __syncthreads();  // the unit's tiles are consumed before the next unit's loads
    }
    if (lane == 0 && a.n_eval) atomicAdd(a.n_eval, n_ev * (unsigned long long)(R * P * 32));
    flush_warp(a, wc, blockIdx.x * NW3 + warp, lane);
}

// The tile screen pays only while the threshold is below the first slot's |y_c|^2 (a pair's first-
// slot margin K0 - theta is positive): dense near-ties (random y over several tasks) never get
// there.  Two kernels are launched back to back, the screened one first; each CTA tests the
// threshold at its start and only the matching kernel sweeps (the threshold only falls while the
// screened one runs, so the second then finds it below too and exits).  Separate kernels keep the
// unscreened sweep's code exactly the plain one (sharing one kernel cost it 3-5 %, C3 random y).
template <int NT, bool SCR>
__global__ void __launch_bounds__(Cfg<NT>::NTH, Cfg<NT>::MINB) k_fit3(const __grid_constant__ FitArgs a) {
    __shared__ FitShared<NT> S;
    if constexpr (TSK) {
        __shared__ int s_use;
        if (threadIdx.x == 0) {
            double y2 = 0.0;
            for (int t = 0; t < a.T; ++t) y2 = fmax(y2, a.G[(int64_t)t * a.mp * a.mp + a.m * a.mp + a.m]);
            const double th = a.collect == 1 ? a.theta0 : ord_dec(*(volatile unsigned long long*)a.theta_g);
            s_use = a.tmax != nullptr && th < y2;
        }
        __syncthreads();
        if ((s_use != 0) != SCR) return;
    }
    fit3_sweep<NT, SCR>(a, S);
}

// Same arithmetic as the fit kernel (hoist on (j, k), sweep variable i), one thread per explicit tuple.
__global__ void k_screen3(const __grid_constant__ FitArgs a, const int64_t* __restrict__ tuples, int64_t count,
                          double* __restrict__ out_lb, int32_t* __restrict__ out_flags) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    double lb;
    out_flags[c] = eval_tuple3(a, tuples[3 * c], tuples[3 * c + 1], tuples[3 * c + 2], &lb);
    out_lb[c] = lb;
}

__global__ void __launch_bounds__(128) k_seed_eval3(const __grid_constant__ FitArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= *a.seed_n) return;
    double lb = 0.0, ub = INFINITY;
    const int fl = a.seed_tup[c * kSeedW] >= 0 ? eval_tuple3(a, a.seed_tup[c * kSeedW + 0], a.seed_tup[c * kSeedW + 1], a.seed_tup[c * kSeedW + 2], &lb, &ub) : 0;
    a.seed_ub[c] = (fl == 3 && ub == ub) ? ub : INFINITY;
}

template <int NT>
int launch_nt(const FitArgs& a0, int nsm, cudaStream_t st) {
    using C = Cfg<NT>;
    FitArgs a = a0;
    const unsigned long long rows = (unsigned long long)a.T * a.mp, cols = (unsigned long long)a.mp;
    if (!make_tma_2d(&a.tmJ, a.G, cols, rows, 32, C::IB) || !make_tma_2d(&a.tmK, a.G, cols, rows, C::KSPAN, C::IB) ||
        !make_tma_2d(&a.tmC, a.G, cols, rows, 2, C::IB) || !make_tma_2d(&a.tmH, a.G, cols, rows, 32, C::KSPAN))
        return -1;
    cudaFuncSetAttribute(k_fit3<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit3<NT, false>, C::NTH, C::smem_bytes);
    if (per_sm < 1) per_sm = 1;
    int grid = nsm * per_sm;
    if (a.collect != 1) seed_launch<3, 18>(k_seed_eval3, a, st);
    if (TSK && a.tmax) {
        k_tile_max<C::IB><<<dim3((unsigned)((a.m + 256) / 256), (unsigned)((a.m + C::IB - 1) / C::IB)), 256, 0, st>>>(
            a.G, a.iforce, a.m, a.mp, a.T, a.tmax);
        cudaFuncSetAttribute(k_fit3<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes);
        k_fit3<NT, true><<<grid, C::NTH, C::smem_bytes, st>>>(a);
    }
    k_fit3<NT, false><<<grid, C::NTH, C::smem_bytes, st>>>(a);
    return grid;
}

}  // namespace

void launch_screen3(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st) {
    if (count > 0) k_screen3<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(a, tuples, count, out_lb, out_flags);
}

// More tasks than the sweep's 8 slots: the slots hold the 8 tasks of largest |y_c|^2, whose bound
// terms alone bound the pooled SSR from below (every task's SSR is >= 0); the slow path, the
// certificates and the exact refit take every task.
int fit3_max_tasks() { return 1 << 16; }
int64_t fit3_tmax_doubles(int64_t m, int64_t mp) {
    (void)mp;
    return TSK ? (m + 1 + (m + 31) / 32) * ((m + 15) / 16) + 1 : 0;  // tile heights >= 16
}
int fit_slots_per_cta() { return NW; }
int fit3_slots_per_cta(int T) {
    return T == 1 ? Cfg<1>::NW : (T == 2 ? Cfg<2>::NW : (T <= 4 ? Cfg<4>::NW : Cfg<8>::NW));
}
int fit3_kspan(int T) {
    switch (T) {
        case 1: return Cfg<1>::KSPAN;
        case 2: return Cfg<2>::KSPAN;
        case 3: return Cfg<3>::KSPAN;
        case 4: return Cfg<4>::KSPAN;
        default: return Cfg<8>::KSPAN;
    }
}
int fit3_grid(int T, int nsm) {
    int per_sm = 0;
    switch (T) {
#define OCC(NT)                                                                                              \
    case NT:                                                                                                 \
        cudaFuncSetAttribute(k_fit3<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<NT>::smem_bytes); \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit3<NT, false>, Cfg<NT>::NTH, Cfg<NT>::smem_bytes); \
        break;
        OCC(1) OCC(2) OCC(3) OCC(4) OCC(5) OCC(6) OCC(7) OCC(8)
#undef OCC
        default:
            if (T < 1) return -1;
            cudaFuncSetAttribute(k_fit3<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<8>::smem_bytes);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit3<8, false>, Cfg<8>::NTH, Cfg<8>::smem_bytes);
    }
    return nsm * (per_sm < 1 ? 1 : per_sm);
}

int fit3_launch(const FitArgs& a, int nsm, cudaStream_t st) {
    switch (a.T) {
        case 1: return launch_nt<1>(a, nsm, st);
        case 2: return launch_nt<2>(a, nsm, st);
        case 3: return launch_nt<3>(a, nsm, st);
        case 4: return launch_nt<4>(a, nsm, st);
        case 5: return launch_nt<5>(a, nsm, st);
        case 6: return launch_nt<6>(a, nsm, st);
        case 7: return launch_nt<7>(a, nsm, st);
        case 8: return launch_nt<8>(a, nsm, st);
        default: return a.T > 8 ? launch_nt<8>(a, nsm, st) : -1;  // T > 8: 8 tasks bound the sweep
    }
}

// Unit table for n = 3: (j-block of 32, k-span, i range), i < j < k < m.
std::vector<int4> fit3_units(int64_t m, int T, int64_t N_total, const std::vector<int64_t>& c2_prefix,
                             int64_t rank_lo, int64_t rank_hi, bool tunable) {
    const int kspan = fit3_kspan(T);
    // i rows per unit: amortizes the (j, k) hoist; L0S_ICH overrides (tuning, single searches
    // only: search parts on different ranks must build identical tables)
    static const int ich_env = [] {
        const char* e = getenv("L0S_ICH");
        const int v = e ? atoi(e) : 0;
        return v > 0 ? v : 4096;
    }();
    const int ich = tunable ? ich_env : 4096;
    std::vector<int4> units;
    int nJ = (int)((m + 31) / 32);
    int nK = (int)((m + kspan - 1) / kspan);
    // first indices c0 whose rank blocks [c2_prefix[c0], c2_prefix[c0+1]) meet [rank_lo, rank_hi)
    int i_first = 0, i_last = (int)m - 1;
    while (i_first < m && c2_prefix[i_first + 1] <= rank_lo) ++i_first;
    while (i_last > 0 && c2_prefix[i_last] >= rank_hi) --i_last;
    for (int jb = 0; jb < nJ; ++jb) {
        int jlo = jb * 32;
        int i_end = (int)std::min<int64_t>(jlo + 31, m - 2);  // largest useful i is < max j
        i_end = std::min(i_end, i_last + 1);
        if (i_end <= i_first) continue;
        for (int kb = jlo / kspan; kb < nK; ++kb) {
            if ((int64_t)kb * kspan + kspan - 1 <= jlo) continue;  // every k <= every j
            for (int lo = i_first; lo < i_end; lo += ich) {
                int hi = std::min(lo + ich, i_end);
                // rank interval of tuples whose first index lies in [lo, hi): prefix sums of C(m-1-v, 2)
                int64_t rmin = c2_prefix[lo], rmax = c2_prefix[hi];
                if (rmax <= rank_lo || rmin >= rank_hi) continue;
                units.push_back(make_int4(jb, kb, lo, hi));
            }
        }
    }
    std::stable_sort(units.begin(), units.end(),
                     [](const int4& x, const int4& y) { return (x.w - x.z) > (y.w - y.z); });
    (void)N_total;
    return units;
}

}  // namespace l0s
