// fitcommon.cuh -- machinery shared by the screened fit kernels (fit3.cu, fit4.cu):
// the error model, the rank-rule certificate, the per-warp top-K' candidate
// buffer and the deferred slow path.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace l0s {
namespace fit {

constexpr int NW = 8;                 // warps per CTA
#ifndef L0S_CAP
#define L0S_CAP 256
#endif
constexpr int CAP = L0S_CAP;          // per-warp candidate buffer (K' <= CAP - 32)
// dimension >= 4 sweeps (one CTA per SM, shared memory to spare) keep longer lists: dense near-
// ties among the keep best (C4: ~260 tuples within the margin of the 10th score) then certify
// in one sweep instead of two
constexpr int CAP_WIDE = 512;
static_assert((CAP & (CAP - 1)) == 0, "warp_sort is a bitonic network over CAP entries");
constexpr double FO_LIM = 1e-3;       // first-order validity: (eta + gam rho)(1 + n tr) <= FO_LIM
constexpr double RANK_SLACK = 1.01;   // safety factor on the rank-rule certificate
constexpr double LOOSE = 1e-3;        // bounds looser than this fraction of |y_c|^2 go to the exact kernel
constexpr double LOOSE32 = 3e-2;      // the same for precision="fp32" (its rounding model is 2^29 x coarser)

// Error model, one task, n features, tr = trace of the inverse of the
// normalized n x n block, tr <= trh + (1 + trh)/d (trh: hoisted (n-1) x (n-1) block):
//   |ssr_gram - ssr_true| <= 2 eta Y2 (1 + n tr)
//   |ssr_ref  - ssr_true| <= 4 gam |y_c||y| + 2 gam rho Y2 (1 + n tr)
// so ssr_ref >= ssr_gram - A - B/d with K = 2 (eta + gam rho),
//   A = 4 gam |y_c| |y| + K Y2 (1 + n trh),   B = n K Y2 (1 + trh)
// valid while vk (1 + n tr) <= FO_LIM.  (|y_c| = sqrt(Y2), |y| = yn: a per-task constant; the
// product matters for a property with a large mean, |y| >> |y_c|, and for fp32's larger gam.)
__device__ __forceinline__ void task_bound(int n, double eta, double gam, double rho, double Y2, double yn,
                                           double trh, double& A, double& B, double& vk) {
    vk = eta + gam * rho;
    const double K = 2.0 * vk;
    A = 4.0 * gam * sqrt(Y2) * yn + K * Y2 * (1.0 + n * trh);
    B = n * K * Y2 * (1.0 + trh);
}

// The same with the pair-independent term precomputed: A0 = 4 gam |y_c| |y|.
__device__ __forceinline__ void task_bound_a0(int n, double eta, double gam, double rho, double Y2, double A0,
                                              double trh, double& A, double& B, double& vk) {
    vk = eta + gam * rho;
    const double K = 2.0 * vk;
    A = A0 + K * Y2 * (1.0 + n * trh);
    B = n * K * Y2 * (1.0 + trh);
}

// Householder QR columnwise backward-error constant for r rows, n features + intercept + rhs,
// with the inner products' rounding bounded probabilistically: |error| <= lambda sqrt(r) u
// with probability >= 1 - 2 exp(-lambda^2 (1-u)^2 / 2) per inner product (Higham & Mary,
// SIAM J. Sci. Comput. 41(5), 2019); lambda = 8 puts the failure probability below 1e-13.
// (The worst-case r u growth would make every feature whose mean/std ratio exceeds ~1e6
// uncertifiable at r = 5000, although the reference's actual error there is ~1e-7.)
//
// precision="fp32" (numba's mixed typing, lsq.py:61-110 on float32 data): every product is
// rounded to float32 (relative 2^-24 per term, no growth with r because the sums run in
// float64) and every stored reflection result is rounded to float32 once per step, so the
// columnwise backward error is O((n+2) u32) plus the float64 accumulation term.
__device__ __host__ __forceinline__ double ref_gamma(double rows, int n, bool fp32 = false) {
    return fp32 ? 2.0 * 8.0 * (n + 2) * (kEps32 + sqrt(rows + 1.0) * kEps)
                : 2.0 * 8.0 * sqrt(rows + 1.0) * (n + 2) * kEps;
}

// 1/d without the IEEE-division subroutine call: MUFU seed + two Newton steps (a few ulp,
// inside the eta slack).  Garbage for d <= 0, which every caller rejects separately.
__device__ __forceinline__ double rcp_newton(double d) {
    double r = rcp_fast_pos(d);
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// Sufficient condition for the reference's rank rule |R_jj| >= tol max|R_jj| (lsq.py:96-101)
// on the uncentered columns [f_1 .. f_n, 1] of one task:
//   every R_jj^2 >= sigma_min([F, 1])^2 >= min(min_f |f_c|^2 / tr, r) / (1 + |mu|)^2,
//   max R_jj^2 <= max(max_f |f|^2, r),  (1 + |mu|)^2 <= 2 (1 + sum_f mean_f^2),
// tr = trace(C^-1) >= 1/lambda_min(C) carrying <= FO_LIM relative error.
template <int N>
__device__ __forceinline__ bool rank_certain(const FitArgs& a, int t, const int64_t (&f)[N], double tr) {
    const int64_t m = a.m;
    const double* qt = a.qf + (int64_t)t * m;
    const double* ut = a.un2 + (int64_t)t * m;
    const double rt = a.rowsd[t];
    double fc_min = INFINITY, mean2 = 0.0, hi = rt;
#pragma unroll
    for (int x = 0; x < N; ++x) {
        const double u = ut[f[x]], q = qt[f[x]];
        fc_min = fmin(fc_min, u * q);
        mean2 += u * (1.0 - q);
        hi = fmax(hi, u);
    }
    const double lo = fmin(fc_min / (tr * (1.0 + 4.0 * FO_LIM)), rt) / (2.0 * (1.0 + mean2 / rt));
    const double tl = sqrt(a.tol2) + 4.0 * ref_gamma(rt, N, a.ref_fp32);  // the reference's rounding of R
    return lo >= tl * tl * hi * RANK_SLACK;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ bool cand_gt(double a, int64_t ra, double b, int64_t rb) {
    return a > b || (a == b && ra > rb);
}

// Warp-wide bitonic sort of the cap-entry buffer by (lb, rank); entries [cnt, cap) are padding.
__device__ __forceinline__ void warp_sort(double* lb, int64_t* rk, int cnt, int lane, int cap) {
    for (int x = cnt + lane; x < cap; x += 32) {
        lb[x] = __longlong_as_double(0x7ff0000000000000ll);
        rk[x] = 0x7fffffffffffffffll;
    }
    __syncwarp();
    for (int k = 2; k <= cap; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int x = lane; x < cap; x += 32) {
                int y = x ^ jj;
                if (y > x) {
                    bool up = (x & k) == 0;
                    double p = lb[x], q = lb[y];
                    int64_t rp = rk[x], rq = rk[y];
                    if (cand_gt(p, rp, q, rq) == up) {
                        lb[x] = q;
                        lb[y] = p;
                        rk[x] = rq;
                        rk[y] = rp;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Per-warp candidate state (shared-memory buffer + warp-uniform count and threshold).
struct WarpCands {
    double* lb;
    int64_t* rk;
    int cnt;
    double theta;
    int counted;  // entries [0, counted) are already in the global histogram
    int cap = CAP;  // buffer entries (a power of two; K' <= cap - 32)
};

// ---- global lower-bound histogram (the shared threshold) ----
// A warp sees ~1/1000 of the tuples, so its own K'-th bound is far looser than the global
// K'-th.  Every tuple a warp keeps (lb below its threshold) is counted once in a global
// histogram of lb (HIST_SUB sub-bins per binary exponent, HIST_EXP exponents below the
// total |y|^2); the upper edge of the first bin at which the cumulative count reaches K' is
// a valid shared threshold: at least K' distinct tuples have smaller bounds, and every tuple
// below it was kept somewhere (all thresholds stay above it).

// bin of a bound (-1: above the histogram's range, not counted -- undercounting is safe)
__device__ __forceinline__ int hist_bin(double lb, int base) {
    if (!(lb > 0.0)) return 0;
    const int b = (int)((unsigned long long)__double_as_longlong(lb) >> (52 - HIST_SUB_BITS)) - base;
    return b < 0 ? 0 : (b >= HIST_BINS ? -1 : b);
}
__device__ __forceinline__ double hist_upper(int b, int base) {
    return __longlong_as_double((long long)((unsigned long long)(base + b + 1) << (52 - HIST_SUB_BITS)));
}

// Count the warp's entries [counted, cnt) (one aggregated atomic per distinct bin per round).
__device__ __forceinline__ void hist_count(const FitArgs& a, WarpCands& wc, int lane) {
    for (int x0 = wc.counted; x0 < wc.cnt; x0 += 32) {
        const int x = x0 + lane;
        const bool on = x < wc.cnt;
        int b = on ? hist_bin(wc.lb[x], a.hist_base) : -1;
        if (b < 0) b = -1 - lane;  // not counted: a key no other lane shares
        const unsigned peers = __match_any_sync(L0S_FULL, b);
        if (b >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(a.hist + b, (unsigned)__popc(peers));
    }
    wc.counted = wc.cnt;
}

// Smallest histogram edge with >= kc counted bounds below it (+inf when fewer).
__device__ __forceinline__ double hist_theta(const FitArgs& a, int lane) {
    constexpr int PER = HIST_BINS / 32;
    static_assert(PER % 4 == 0, "each lane's bins load as uint4");
    const unsigned* h = a.hist + lane * PER;
    unsigned sum = 0;
#pragma unroll
    for (int x = 0; x < PER; x += 4) {  // 16-byte loads: a quarter of the strided transactions
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(h + x));
        sum += v.x + v.y + v.z + v.w;
    }
    unsigned inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(L0S_FULL, inc, o);
        if (lane >= o) inc += v;
    }
    const unsigned hit = __ballot_sync(L0S_FULL, inc >= (unsigned)a.kc);
    if (!hit) return INFINITY;
    const int L = __ffs(hit) - 1;
    // lane L's bins again, spread over the warp (two per lane) and scanned: the first bin where the
    // running count reaches kc (counts only grow, so the re-read total still reaches it)
    static_assert(PER <= 64, "two bins per lane");
    const unsigned before = __shfl_sync(L0S_FULL, inc - sum, L);
    const unsigned* hL = a.hist + L * PER;
    unsigned s0 = lane < PER ? __ldcg(hL + lane) : 0u;
    unsigned s1 = lane + 32 < PER ? __ldcg(hL + 32 + lane) : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned v0 = __shfl_up_sync(L0S_FULL, s0, o), v1 = __shfl_up_sync(L0S_FULL, s1, o);
        if (lane >= o) {
            s0 += v0;
            s1 += v1;
        }
    }
    s1 += __shfl_sync(L0S_FULL, s0, 31);
    const unsigned h0 = __ballot_sync(L0S_FULL, before + s0 >= (unsigned)a.kc);
    const unsigned h1 = __ballot_sync(L0S_FULL, lane + 32 < PER && before + s1 >= (unsigned)a.kc);
    if (h0) return hist_upper(L * PER + __ffs(h0) - 1, a.hist_base);
    if (h1) return hist_upper(L * PER + 32 + __ffs(h1) - 1, a.hist_base);
    return INFINITY;
}

// Collect modes: append the warp's buffer to the global candidate list (collect == 2, the
// histogram-threshold mode of large keep: only the entries still below the warp's threshold;
// the others are above the final threshold too).
__device__ __forceinline__ void flush_collect(const FitArgs& a, WarpCands& wc, int lane) {
    const unsigned lt = lanemask_lt();
    for (int x0 = 0; x0 < wc.cnt; x0 += 32) {
        const int x = x0 + lane;
        const bool on = x < wc.cnt && (a.collect == 1 || wc.lb[x] < wc.theta);
        const unsigned bal = __ballot_sync(L0S_FULL, on);
        unsigned long long b0 = 0;
        if (lane == 0 && bal) b0 = atomicAdd(a.coll_cnt, (unsigned long long)__popc(bal));
        b0 = __shfl_sync(L0S_FULL, b0, 0);
        if (on) {
            const unsigned long long idx = b0 + __popc(bal & lt);
            if ((int64_t)idx < a.coll_cap) {
                a.coll_lb[idx] = wc.lb[x];
                a.coll_rank[idx] = wc.rk[x];
            }
        }
    }
    wc.cnt = 0;
    wc.counted = 0;
    __syncwarp();
}

// Deferred slow path: drain the pending bits (one tuple per lane per round).
//   eval(b, &lb, &rank) -> 0 drop, 1 insert (lb < theta checked here), 2 exact kernel
//   on_theta()          -> called after the warp's threshold dropped (refresh hoisted constants)
template <int NPW, typename Eval, typename OnTheta>
__device__ __forceinline__ void drain_pending(const FitArgs& a, unsigned (&pend)[NPW], WarpCands& wc, int lane,
                                              Eval eval, OnTheta on_theta) {
    const unsigned lt = lanemask_lt();
    for (;;) {
        int b = -1;
#pragma unroll
        for (int w = 0; w < NPW; ++w)
            if (b < 0 && pend[w]) {
                b = w * 32 + __ffs(pend[w]) - 1;
                pend[w] &= pend[w] - 1u;
            }
        if (!__any_sync(L0S_FULL, b >= 0)) break;
        int kind = 0;
        double lbv = 0.0;
        int64_t rkv = 0;
        if (b >= 0) {
            kind = eval(b, &lbv, &rkv);
            if (kind == 1 && !(lbv < wc.theta)) kind = 0;
        }
        const unsigned im = __ballot_sync(L0S_FULL, kind == 1);
        if (im) {
            if (kind == 1) {
                const int pos = wc.cnt + __popc(im & lt);
                wc.lb[pos] = lbv;
                wc.rk[pos] = rkv;
            }
            wc.cnt += __popc(im);
            if (a.collect != 1) {
                // count the new entries in the global histogram right away (the shared
                // threshold must not wait for this warp's buffer to fill)
                int hb = (kind == 1) ? hist_bin(lbv, a.hist_base) : -1;
                if (hb < 0) hb = -1 - lane;
                const unsigned peers = __match_any_sync(L0S_FULL, hb);
                if (hb >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(a.hist + hb, (unsigned)__popc(peers));
                wc.counted = wc.cnt;
            }
        }
        const unsigned il = __ballot_sync(L0S_FULL, kind == 2);
        if (il) {
            unsigned long long b0 = 0;
            const int leader = __ffs(il) - 1;
            if (lane == leader) b0 = atomicAdd(a.ill_cnt, (unsigned long long)__popc(il));
            b0 = __shfl_sync(L0S_FULL, b0, leader);
            if (kind == 2) {
                const unsigned long long idx = b0 + __popc(il & lt);
                if ((int64_t)idx < a.ill_cap) a.ill[idx] = rkv;
            }
        }
        __syncwarp();
        if (wc.cnt > wc.cap - 32) {
            if (a.collect) {
                flush_collect(a, wc, lane);
                if (a.collect == 2) {
                    // histogram threshold (large keep): the K'-th smallest bound counted anywhere
                    const double th = fmin(hist_theta(a, lane), ord_dec(*(volatile unsigned long long*)a.theta_g));
                    if (th < wc.theta) {
                        wc.theta = th;
                        if (lane == 0) atomicMin(a.theta_g, ord_enc(wc.theta));
                        on_theta();
                    }
                    __syncwarp();
                }
            } else {
                hist_count(a, wc, lane);
                warp_sort(wc.lb, wc.rk, wc.cnt, lane, wc.cap);
                if (wc.cnt > a.kc) wc.cnt = a.kc;
                wc.counted = wc.cnt;
                double th = hist_theta(a, lane);
                if (wc.cnt == a.kc) th = fmin(th, wc.lb[a.kc - 1]);
                th = fmin(th, ord_dec(*(volatile unsigned long long*)a.theta_g));
                if (th < wc.theta) {
                    wc.theta = th;
                    if (lane == 0) atomicMin(a.theta_g, ord_enc(wc.theta));
                    on_theta();
                }
                __syncwarp();
            }
        }
    }
}

// Seed of the shared threshold (one CTA of 256 threads, launched before the sweep): the F
// features with the largest pooled single-feature explained variance sum_t c_f^2, and every
// N-subset of them inside the rank range is evaluated with the Gram bound pair (lb, ub).  The
// kc-th smallest upper bound among the certified subsets is >= the kc-th smallest lower bound
// over all tuples, so it is a valid starting threshold: the sweep's first tiles then drop the
// hopeless tuples instead of sending every one of them through the slow path.
constexpr int SEED_MAX = 1024;
constexpr int SEED_POOL = 16384;  // candidate features of the seed (dynamic smem doubles)
struct SeedSmem {
    double ub[SEED_MAX];
    short sub[SEED_MAX][kSeedW];
    int top[32];
    double rv[32];
    int ri[32];
    int nsub;
};

// Phase 1: top-F features and their N-subsets (ascending feature order); returns the count
// (0 when fewer than F live features or fewer than kc subsets).
template <int N, int F>
__device__ int seed_subsets(const FitArgs& a, SeedSmem& S) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t m = a.m, mp = a.mp;
    if (m < F) return 0;
    // pooled single-feature scores of the first SEED_POOL features, once, into shared memory
    // (dynamic, SEED_POOL doubles); the F selection rounds then only scan shared memory
    extern __shared__ double s_score[];
    const int pool = (int)(m < SEED_POOL ? m : SEED_POOL);
    for (int f = tid; f < pool; f += blockDim.x) {
        double sc = 0.0;
        for (int t = 0; t < a.T; ++t) {
            const double c = a.G[(int64_t)t * mp * mp + m * mp + f];
            sc = fma(c, c, sc);
        }
        s_score[f] = sc;  // NaN (dead feature) never wins a comparison
    }
    __syncthreads();
    for (int r = 0; r < F; ++r) {
        double best = -1.0;
        int bi = -1;
        for (int f = tid; f < pool; f += blockDim.x)
            if (s_score[f] > best) {
                best = s_score[f];
                bi = f;
            }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(L0S_FULL, best, o);
            const int oi = __shfl_down_sync(L0S_FULL, bi, o);
            if (ov > best) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            S.rv[warp] = best;
            S.ri[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (S.rv[w] > S.rv[0]) {
                    S.rv[0] = S.rv[w];
                    S.ri[0] = S.ri[w];
                }
            S.top[r] = S.ri[0];
            if (S.ri[0] >= 0) s_score[S.ri[0]] = -1.0;  // taken
        }
        __syncthreads();
    }
    // subsets of the F winners (ascending feature order), enumerated in parallel: thread c
    // unranks c in the lexicographic order of C(F, N)
    if (tid == 0) {
        bool ok = true;
        for (int r = 0; r < F; ++r) ok &= S.top[r] >= 0;  // fewer than F live features: no seed
        for (int x = 1; ok && x < F; ++x)
            for (int z = x; z > 0 && S.top[z] < S.top[z - 1]; --z) {
                const int q = S.top[z];
                S.top[z] = S.top[z - 1];
                S.top[z - 1] = q;
            }
        int total = 1;  // C(F, N)
        for (int x = 0; x < N; ++x) total = total * (F - x) / (x + 1);
        total = total < SEED_MAX ? total : SEED_MAX;
        S.nsub = (ok && total >= a.kc) ? total : 0;
    }
    __syncthreads();
    for (int c = tid; c < S.nsub; c += blockDim.x) {
        int r = c, e = 0;
        for (int x = 0; x < N; ++x) {
            const int rem = N - 1 - x;
            for (;;) {
                int blk = 1;  // C(F - 1 - e, rem)
                for (int z = 0; z < rem; ++z) blk = blk * (F - 1 - e - z) / (z + 1);
                if (r < blk) break;
                r -= blk;
                ++e;
            }
            S.sub[c][x] = (short)e;
            ++e;
        }
    }
    __syncthreads();
    return S.nsub;
}

// Subset c's features and whether its rank lies in the searched range.
template <int N>
__device__ __forceinline__ bool seed_tuple(const FitArgs& a, const SeedSmem& S, int c, int64_t (&f)[N]) {
    const int64_t m = a.m;
    int64_t rk = a.N_total - 1;
    for (int x = 0; x < N; ++x) {
        f[x] = S.top[S.sub[c][x]];
        rk -= a.binom[(int64_t)(N - x) * (m + 1) + (m - 1 - f[x])];
    }
    return !a.ranged || (rk >= a.rank_lo && rk < a.rank_hi);
}

namespace {
// Row-block maxima for the tile screen (TSK), blocks of IB rows (the sweep's tile height,
// aligned at row 0) of the first task slot (the task of largest |y_c|^2, first on ties, as k_fit3
// orders them; k_fit4 screens the same task): [col][block] max |C[i, col]| over i != col for col <= m (col = m: max |c_i|;
// the diagonal is left out -- every tile that reaches a lane's own j or k would fail), then
// [j-block][block] the maximum over the j-block's 32 columns, then the slot's task index.  +inf
// where a row is iforce-flagged (column m) or an entry is NaN.  One read of one task's Gram.
template <int IB>
__global__ void __launch_bounds__(256) k_tile_max(const double* __restrict__ G, const unsigned char* __restrict__ iforce,
                                                  int64_t m, int64_t mp, int T, double* __restrict__ out) {
    __shared__ int s_t0;
    const int64_t nbk = (m + IB - 1) / IB, nJ = (m + 31) / 32;
    if (threadIdx.x == 0) {
        int best = 0;
        double bv = G[m * mp + m];
        for (int t = 1; t < T; ++t) {
            const double v = G[(int64_t)t * mp * mp + m * mp + m];
            if (v > bv) {
                bv = v;
                best = t;
            }
        }
        s_t0 = best;
        if (blockIdx.x == 0 && blockIdx.y == 0) out[(m + 1 + nJ) * nbk] = (double)best;
    }
    __syncthreads();
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    const double* Gt = G + (int64_t)s_t0 * mp * mp;
    double mx = 0.0;
    if (col <= m) {
        bool bad = false;
        for (int64_t i = b * IB; i < min(b * IB + IB, m); ++i) {
            if (i == col) continue;  // C_jj = 1: a tuple never repeats a feature (i < j < k ...)
            const double v = Gt[i * mp + col];
            bad |= (v != v) || (col == m && iforce[i]);
            mx = fmax(mx, fabs(v));
        }
        if (bad) mx = INFINITY;
        out[col * nbk + b] = mx;
    }
    double jm = col < m ? mx : 0.0;  // warps cover whole j-blocks (blockDim and the x offset are multiples of 32)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) jm = fmax(jm, __shfl_xor_sync(L0S_FULL, jm, o));
    if ((threadIdx.x & 31) == 0 && col < m) out[(m + 1) * nbk + (col >> 5) * nbk + b] = jm;
}

// Seed phase 1 (one CTA of 512): the subsets, written to a.seed_tup (-1: outside the rank range).
template <int N, int F>
__global__ void __launch_bounds__(512, 1) k_seed_select(const __grid_constant__ FitArgs a) {
    __shared__ SeedSmem S;
    const int ns = seed_subsets<N, F>(a, S);
    for (int c = threadIdx.x; c < ns; c += blockDim.x) {
        int64_t f[N];
        const bool in = seed_tuple<N>(a, S, c, f);
        for (int x = 0; x < N; ++x) a.seed_tup[c * kSeedW + x] = in ? f[x] : -1;
    }
    if (threadIdx.x == 0) *a.seed_n = ns;
}

// Seed phase 3 (one CTA of 512): the kc-th smallest upper bound becomes the starting threshold
// (bitonic sort of the <= SEED_MAX bounds in shared memory).
__global__ void __launch_bounds__(512, 1) k_seed_commit(const __grid_constant__ FitArgs a) {
    __shared__ double ub[SEED_MAX];
    const int ns = *a.seed_n;
    if (ns < a.kc) return;
    for (int c = threadIdx.x; c < SEED_MAX; c += blockDim.x) ub[c] = c < ns ? a.seed_ub[c] : INFINITY;
    __syncthreads();
    for (int k = 2; k <= SEED_MAX; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int x = threadIdx.x; x < SEED_MAX; x += blockDim.x) {
                const int y = x ^ jj;
                if (y > x) {
                    const double p = ub[x], q = ub[y];
                    const bool up = (x & k) == 0;
                    if ((p > q) == up) {
                        ub[x] = q;
                        ub[y] = p;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0) {
        const double v = ub[a.kc - 1];
        // >= keep tuples score at most the keep-th bound: caps the global keep-th score (search
        // parts, api.cu)
        // (only when keep <= kc: the kc-th bound guarantees kc tuples below it, not keep)
        if (a.seed_cap) *a.seed_cap = (a.keep >= 1 && a.keep <= a.kc) ? ub[a.keep - 1] : INFINITY;
        if (v < INFINITY) {
            const double th = v + fabs(v) * 1e-9 + 1e-300;  // strictly above kc certified bounds
            atomicMin(a.theta_g, ord_enc(th));
        }
    }
}
}  // namespace

// Phase 2 is the dimension's own eval kernel (one thread per subset, grid over SEED_MAX):
//   k_seed_evalN: a.seed_ub[c] = upper bound of subset c if certified, else +inf.
template <int N, int F, typename E>
inline void seed_launch(E eval_kernel, const FitArgs& a, cudaStream_t st) {
    const int bytes = (int)(sizeof(double) * (a.m < SEED_POOL ? a.m : SEED_POOL));
    cudaFuncSetAttribute(k_seed_select<N, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    k_seed_select<N, F><<<1, 512, bytes, st>>>(a);
    eval_kernel<<<SEED_MAX / 128, 128, 0, st>>>(a);
    k_seed_commit<<<1, 512, 0, st>>>(a);
}

// End of the persistent loop: write the warp's list (or flush the collect buffer).
__device__ __forceinline__ void flush_warp(const FitArgs& a, WarpCands& wc, int slot, int lane) {
    if (a.collect) {
        flush_collect(a, wc, lane);
        if (lane == 0) a.wl_cnt[slot] = 0;
    } else {
        warp_sort(wc.lb, wc.rk, wc.cnt, lane, wc.cap);
        if (wc.cnt > a.kc) wc.cnt = a.kc;
        for (int x = lane; x < wc.cnt; x += 32) {
            a.wl_lb[(int64_t)slot * a.kc + x] = wc.lb[x];
            a.wl_rank[(int64_t)slot * a.kc + x] = wc.rk[x];
        }
        if (lane == 0) {
            a.wl_cnt[slot] = wc.cnt;
            if (wc.cnt == a.kc) atomicMin(a.theta_g, ord_enc(wc.lb[a.kc - 1]));
        }
    }
}

}  // namespace fit
}  // namespace l0s
