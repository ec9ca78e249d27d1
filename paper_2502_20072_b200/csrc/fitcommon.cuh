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
constexpr double FO_LIM = 1e-3;       // first-order validity: (eta + gam rho)(1 + n tr) <= FO_LIM
constexpr double RANK_SLACK = 1.01;   // safety factor on the rank-rule certificate
constexpr double LOOSE = 1e-3;        // bounds looser than this fraction of |y_c|^2 go to the exact kernel

// Error model, one task, n features, tr = trace of the inverse of the
// normalized n x n block, tr <= trh + (1 + trh)/d (trh: hoisted (n-1) x (n-1) block):
//   |ssr_gram - ssr_true| <= 2 eta Y2 (1 + n tr)
//   |ssr_ref  - ssr_true| <= 4 gam |y_c||y| + 2 gam rho Y2 (1 + n tr)
// so ssr_ref >= ssr_gram - A - B/d with K = 2 (eta + gam rho),
//   A = 2 gam (|y_c|^2 + |y|^2) + K Y2 (1 + n trh),   B = n K Y2 (1 + trh)
// (4ab <= 2(a^2 + b^2) removes the square root), valid while vk (1 + n tr) <= FO_LIM.
__device__ __forceinline__ void task_bound(int n, double eta, double gam, double rho, double Y2, double yn,
                                           double trh, double& A, double& B, double& vk) {
    vk = eta + gam * rho;
    const double K = 2.0 * vk;
    A = 2.0 * gam * (Y2 + yn * yn) + K * Y2 * (1.0 + n * trh);
    B = n * K * Y2 * (1.0 + trh);
}

// Householder QR columnwise backward-error constant for r rows, n features + intercept + rhs,
// with the inner products' rounding bounded probabilistically: |error| <= lambda sqrt(r) u
// with probability >= 1 - 2 exp(-lambda^2 (1-u)^2 / 2) per inner product (Higham & Mary,
// SIAM J. Sci. Comput. 41(5), 2019); lambda = 8 puts the failure probability below 1e-13.
// (The worst-case r u growth would make every feature whose mean/std ratio exceeds ~1e6
// uncertifiable at r = 5000, although the reference's actual error there is ~1e-7.)
__device__ __host__ __forceinline__ double ref_gamma(double rows, int n) {
    return 2.0 * 8.0 * sqrt(rows + 1.0) * (n + 2) * kEps;
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
    const double tl = sqrt(a.tol2) + 4.0 * ref_gamma(rt, N);  // the reference's rounding of R
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

// Warp-wide bitonic sort of the CAP-entry buffer by (lb, rank); entries [cnt, CAP) are padding.
__device__ __forceinline__ void warp_sort(double* lb, int64_t* rk, int cnt, int lane) {
    for (int x = cnt + lane; x < CAP; x += 32) {
        lb[x] = __longlong_as_double(0x7ff0000000000000ll);
        rk[x] = 0x7fffffffffffffffll;
    }
    __syncwarp();
    for (int k = 2; k <= CAP; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int x = lane; x < CAP; x += 32) {
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
};

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
        if (wc.cnt > CAP - 32) {
            if (a.collect) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(a.coll_cnt, (unsigned long long)wc.cnt);
                b0 = __shfl_sync(L0S_FULL, b0, 0);
                for (int x = lane; x < wc.cnt; x += 32)
                    if ((int64_t)(b0 + x) < a.coll_cap) {
                        a.coll_lb[b0 + x] = wc.lb[x];
                        a.coll_rank[b0 + x] = wc.rk[x];
                    }
                wc.cnt = 0;
                __syncwarp();
            } else {
                warp_sort(wc.lb, wc.rk, wc.cnt, lane);
                if (wc.cnt > a.kc) wc.cnt = a.kc;
                if (wc.cnt == a.kc && wc.lb[a.kc - 1] < wc.theta) {
                    wc.theta = wc.lb[a.kc - 1];
                    if (lane == 0) atomicMin(a.theta_g, ord_enc(wc.theta));
                    on_theta();
                }
                __syncwarp();
            }
        }
    }
}

// End of the persistent loop: write the warp's list (or flush the collect buffer).
__device__ __forceinline__ void flush_warp(const FitArgs& a, WarpCands& wc, int slot, int lane) {
    if (a.collect) {
        unsigned long long b0 = 0;
        if (lane == 0 && wc.cnt > 0) b0 = atomicAdd(a.coll_cnt, (unsigned long long)wc.cnt);
        b0 = __shfl_sync(L0S_FULL, b0, 0);
        for (int x = lane; x < wc.cnt; x += 32)
            if ((int64_t)(b0 + x) < a.coll_cap) {
                a.coll_lb[b0 + x] = wc.lb[x];
                a.coll_rank[b0 + x] = wc.rk[x];
            }
        if (lane == 0) a.wl_cnt[slot] = 0;
    } else {
        warp_sort(wc.lb, wc.rk, wc.cnt, lane);
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
