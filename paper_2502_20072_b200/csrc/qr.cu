// qr.cu -- QR screen for the tuples the Gram screen cannot certify (near-collinear
// features, features nearly collinear with the intercept).
//
// One warp per (tuple, task) system [f_c0 .. f_c(n-1), 1 | y] (the reference's column
// order, lsq.py:141-147).  Every lane folds its rows (i = lane, lane+32, ...) into a
// register-resident upper-triangular R with Givens rotations, then the 32 triangles are
// merged pairwise through warp shuffles (5 levels).  Givens QR is backward stable, and the
// result is the reference's R up to signs and rounding, so
//   ssr   = R[p][p]^2                          (p = n+1, the rhs column)
//   ratio = min_j |R_jj| / max_j |R_jj|, j < p (the rank rule's quantity, lsq.py:96-101)
// carry about eps/ratio relative error; the search refits bit-exactly (exact.cu) every
// accepted tuple whose QR score can reach the top list within that margin (api.cu).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace l0s {
namespace {


// packed upper triangle: row j starts at off(j) = j*NC - j*(j-1)/2
template <int NC>
__device__ __forceinline__ constexpr int off(int j) {
    return j * NC - j * (j - 1) / 2;
}

// Fold row x (entries before `start` are zero) into R by Givens rotations.
template <int NC>
__device__ __forceinline__ void givens_row(double (&R)[NC * (NC + 1) / 2], double (&x)[NC], int start) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        if (j < start) continue;
        const double a = R[off<NC>(j)], b = x[j];
        if (b == 0.0) continue;
        // 1/sqrt(a^2 + b^2): MUFU seed + two Newton steps (full precision, no divide)
        const double q = fma(a, a, b * b);
        double ir;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(ir) : "d"(q));
        ir = ir * fma(-0.5 * q * ir, ir, 1.5);
        ir = ir * fma(-0.5 * q * ir, ir, 1.5);
        const double c = a * ir, s = b * ir;
        R[off<NC>(j)] = q * ir;
#pragma unroll
        for (int k = j + 1; k < NC; ++k) {
            const double rk = R[off<NC>(j) + (k - j)], xk = x[k];
            R[off<NC>(j) + (k - j)] = fma(c, rk, s * xk);
            x[k] = fma(c, xk, -s * rk);
        }
    }
}

// Fold a block of B rows X[b][.] (entries before `start` zero) into R by one structured
// Householder reflection per column: the reflector touches R's row j and the block only.
// B rows share each square root and reciprocal; the dot products are short trees.
template <int NC, int B>
__device__ __forceinline__ void householder_block(double (&R)[NC * (NC + 1) / 2], double (&X)[B][NC], int start) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        if (j < start) continue;
        const double rjj = R[off<NC>(j)];
        double nb = 0.0;
#pragma unroll
        for (int b = 0; b < B; ++b) nb = fma(X[b][j], X[b][j], nb);
        if (nb == 0.0) continue;  // the block is already zero in this column
        const double nrm2 = fma(rjj, rjj, nb);
        double ir;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(ir) : "d"(nrm2));
        ir = ir * fma(-0.5 * nrm2 * ir, ir, 1.5);
        ir = ir * fma(-0.5 * nrm2 * ir, ir, 1.5);
        const double nrm = nrm2 * ir;
        const double alpha = rjj >= 0.0 ? -nrm : nrm;
        const double v0 = rjj - alpha;
        const double vtv = fma(v0, v0, nb);  // = 2 nrm (nrm + |rjj|)
        double iv;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(iv) : "d"(vtv));
        iv = iv * fma(-vtv, iv, 2.0);
        iv = iv * fma(-vtv, iv, 2.0);
        const double f2 = 2.0 * iv;
#pragma unroll
        for (int c = j + 1; c < NC; ++c) {
            double w = v0 * R[off<NC>(j) + (c - j)];
#pragma unroll
            for (int b = 0; b < B; ++b) w = fma(X[b][j], X[b][c], w);
            const double f = w * f2;
            R[off<NC>(j) + (c - j)] = fma(-f, v0, R[off<NC>(j) + (c - j)]);
#pragma unroll
            for (int b = 0; b < B; ++b) X[b][c] = fma(-f, X[b][j], X[b][c]);
        }
        R[off<NC>(j)] = alpha;
    }
}

template <int NC>
__global__ void __launch_bounds__(256) k_qr_warp(QrArgs a) {
    constexpr int NR = NC * (NC + 1) / 2;
    const int lane = threadIdx.x & 31;
    const int64_t g = a.g0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (g >= a.total) return;
    const int64_t tup_i = g / a.T;
    const int task = (int)(g % a.T);
    const int n = NC - 2, p = NC - 1;
    int64_t tup[NC - 2];
    unrank_lex(a.ranks[tup_i], a.m, n, a.binom, tup);
    const int64_t lo = a.bounds[task];
    const int rows = (int)(a.bounds[task + 1] - lo);
    const double* X = a.Xp;
    // lane-local TSQR: blocks of QB rows (rows lane, lane+32, ...) folded into R
    constexpr int QB = 4;
    double R[NR];
#pragma unroll
    for (int e = 0; e < NR; ++e) R[e] = 0.0;
    for (int i0 = lane; i0 < rows; i0 += 32 * QB) {
        double Xb[QB][NC];
#pragma unroll
        for (int b = 0; b < QB; ++b) {
            const int i = i0 + 32 * b;
            const bool in = i < rows;
#pragma unroll
            for (int k = 0; k < NC - 2; ++k) Xb[b][k] = in ? X[tup[k] * a.s + lo + i] : 0.0;
            Xb[b][NC - 2] = in ? 1.0 : 0.0;
            Xb[b][NC - 1] = in ? a.yp[lo + i] : 0.0;
        }
        householder_block<NC, QB>(R, Xb, 0);
    }
    // merge the lanes' triangles: partner rows enter as rows with leading zeros
#pragma unroll
    for (int offs = 16; offs >= 1; offs >>= 1) {
        double P[NR];
#pragma unroll
        for (int e = 0; e < NR; ++e) P[e] = __shfl_down_sync(L0S_FULL, R[e], offs);
        if (lane < offs) {
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                double x[NC];
#pragma unroll
                for (int k = 0; k < NC; ++k) x[k] = (k < j) ? 0.0 : P[off<NC>(j) + (k - j)];
                givens_row<NC>(R, x, j);
            }
        }
    }
    if (lane == 0) {
        double mx = 0.0, mn = INFINITY;
#pragma unroll
        for (int j = 0; j < NC - 1; ++j) {
            const double d = (j < rows) ? fabs(R[off<NC>(j)]) : 0.0;
            mx = fmax(mx, d);
            mn = fmin(mn, d);
        }
        const double rpp = R[off<NC>(p)];
        a.ssr[g] = (rows > p) ? rpp * rpp : 0.0;
        a.ratio[g] = (mx > 0.0) ? mn / mx : 0.0;
    }
}

// pooled score (sum over tasks in order / s) and the worst ratio over tasks
__global__ void k_qr_finalize(QrArgs a, int64_t count) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    double tot = 0.0, rmin = INFINITY;
    for (int t = 0; t < a.T; ++t) {
        tot += a.ssr[c * a.T + t];
        rmin = fmin(rmin, a.ratio[c * a.T + t]);
    }
    a.score[c] = tot / (double)a.s;
    a.min_ratio[c] = rmin;
}

// Device-side selection of the ill tuples that can still reach the top list:
// the reference's rank rule must not certainly reject them, and their QR score minus the QR's
// error margin (~ eps / ratio, with a large safety factor) must not exceed the keep-th score.
__global__ void k_qr_select(const double* __restrict__ score, const double* __restrict__ min_ratio,
                            const int64_t* __restrict__ ranks, int64_t count, double tol, double sk, double yy_s,
                            int64_t* __restrict__ sel, unsigned long long* __restrict__ nsel, int64_t cap) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    const double r = min_ratio[c], sc = score[c];
    if (r < tol * (1.0 - 1e-3)) return;  // the reference's rank rule rejects it in some task
    const double margin = 1e3 * kEps * yy_s / fmax(r, 1e-300) + 1e-9 * fabs(sc);
    if (sc - margin > sk) return;
    const unsigned long long k = atomicAdd(nsel, 1ull);
    if ((int64_t)k < cap) sel[k] = ranks[c];
}

}  // namespace

void launch_qr_finalize(const QrArgs& a, int64_t count, cudaStream_t st, int64_t* launches) {
    if (count > 0) {
        k_qr_finalize<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(a, count);
        if (launches) ++*launches;
    }
}

void launch_qr_select(const double* score, const double* min_ratio, const int64_t* ranks, int64_t count, double tol,
                      double sk, double yy_s, int64_t* sel, unsigned long long* nsel, int64_t cap, cudaStream_t st) {
    if (count > 0)
        k_qr_select<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(score, min_ratio, ranks, count, tol, sk, yy_s, sel,
                                                                       nsel, cap);
}

void launch_qr_screen(const QrArgs& a0, int64_t count, cudaStream_t st, int64_t* launches) {
    QrArgs a = a0;
    a.total = count * a.T;
    const int64_t per_launch = (int64_t)1 << 28;  // warps
    for (int64_t g0 = 0; g0 < a.total; g0 += per_launch) {
        a.g0 = g0;
        const int64_t w = std::min(per_launch, a.total - g0);
        const unsigned blocks = (unsigned)((w + 7) / 8);
        switch (a.n) {
            case 1: k_qr_warp<3><<<blocks, 256, 0, st>>>(a); break;
            case 2: k_qr_warp<4><<<blocks, 256, 0, st>>>(a); break;
            case 3: k_qr_warp<5><<<blocks, 256, 0, st>>>(a); break;
            case 4: k_qr_warp<6><<<blocks, 256, 0, st>>>(a); break;
            case 5: k_qr_warp<7><<<blocks, 256, 0, st>>>(a); break;
            default: k_qr_warp<8><<<blocks, 256, 0, st>>>(a); break;
        }
        if (launches) ++*launches;
    }
    if (count > 0) {
        k_qr_finalize<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(a, count);
        if (launches) ++*launches;
    }
}

}  // namespace l0s
