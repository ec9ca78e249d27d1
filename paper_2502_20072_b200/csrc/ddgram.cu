// ddgram.cu -- the QR screen of many ill-conditioned tuples through a double-double Gram.
//
// The TSQR screen (qr.cu) reads every ill tuple's n + 2 columns and factors them: at C4
// (6.9 M ill tuples, 5000 rows) that is 1.4 TB of L2 reads and 255 ms.  The tuples share their
// columns, so when there are many of them the uncentered Gram of every staged column,
//     H[a][b] = sum_i x_a(i) x_b(i)     rows a: the m features, the property y (row m), the
//                                        intercept's column of ones (row m + 1)
// is formed once per task in double-double (Ogita-Rump-Oishi Dot2: TwoProduct by FMA,
// TwoSum of the products, the errors summed aside; |error| <= eps |H| + gamma_{r}^2 sum |x_a x_b|,
// ~3e-25 relative at r = 5000), and every (tuple, task) is screened by an LDL^T of its
// (n + 2) x (n + 2) block [f_0 .. f_{n-1}, 1 | y] in double-double (the reference's column order,
// lsq.py:141-147): the pivots are R_jj^2 of the reference's QR up to its rounding, so
//   ssr   = d_p (the property's pivot)
//   ratio = sqrt(min_{j<p} d_j / max_{j<p} d_j)   (min |R_jj| / max |R_jj|, lsq.py:96-101)
// with errors far inside the select kernel's margins (api.cu screen_ill):
// the Gram's backward error moves d_j by ~3e-25 |H| / d_j relative, i.e. below 1e-4 for every
// ratio the rank rule keeps (>= 1e-10); a pivot at or below zero means R_jj^2 <= that error,
// ratio 0, a tuple the reference's rank rule rejects.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace l0s {
namespace {

struct dd {
    double hi, lo;
};

// every operation explicitly rounded: no contraction into FMAs across the error-free steps
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double z = __dsub_rn(s, a);
    return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, z)), __dsub_rn(b, z))};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {  // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
    const dd s = two_sum(x.hi, y.hi);
    const dd t = two_sum(x.lo, y.lo);
    dd u = fast_two_sum(s.hi, __dadd_rn(s.lo, t.hi));
    return fast_two_sum(u.hi, __dadd_rn(u.lo, t.lo));
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    const double p = __dmul_rn(x.hi, y.hi);
    const double e = fma(x.hi, y.hi, -p);
    const double t = fma(x.hi, y.lo, fma(x.lo, y.hi, e));
    return fast_two_sum(p, t);
}
__device__ __forceinline__ dd dd_div(dd x, dd y) {
    const double q1 = __ddiv_rn(x.hi, y.hi);
    const dd r = dd_add(x, dd_neg(dd_mul({q1, 0.0}, y)));
    const double q2 = __ddiv_rn(r.hi, y.hi);
    const dd r2 = dd_add(r, dd_neg(dd_mul({q2, 0.0}, y)));
    const double q3 = __ddiv_rn(r2.hi, y.hi);
    const dd q = fast_two_sum(q1, q2);
    return dd_add(q, {q3, 0.0});
}

// ---- the Gram: one CTA per 64 x 64 tile (a-block <= b-block) of one task, 16 x 16 threads of
// 4 x 4 entries, samples staged through shared memory 32 at a time ----
constexpr int DG_T = 64, DG_K = 32;

__device__ __forceinline__ double dd_row_value(const double* Xp, const double* yp, int64_t m, int64_t s, int64_t lo,
                                               int64_t a, int64_t i) {
    if (a < m) return Xp[a * s + lo + i];
    if (a == m) return yp[lo + i];
    return a == m + 1 ? 1.0 : 0.0;
}

__global__ void __launch_bounds__(256) k_ddgram(const double* __restrict__ Xp, const double* __restrict__ yp,
                                               int64_t m, int64_t s, const int64_t* __restrict__ bounds, int64_t LD,
                                               const int2* __restrict__ tiles, double* __restrict__ Hhi,
                                               double* __restrict__ Hlo) {
    __shared__ double sa[DG_K][DG_T + 1], sb[DG_K][DG_T + 1];
    const int t = blockIdx.y;
    const int2 tl = tiles[blockIdx.x];
    const int64_t a0 = (int64_t)tl.x * DG_T, b0 = (int64_t)tl.y * DG_T;
    const int64_t lo = bounds[t], r = bounds[t + 1] - lo;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double sh[4][4], cl[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) sh[u][v] = cl[u][v] = 0.0;
    for (int64_t k0 = 0; k0 < r; k0 += DG_K) {
        __syncthreads();
        for (int x = threadIdx.x; x < DG_K * DG_T; x += 256) {
            const int row = x / DG_K, k = x % DG_K;  // consecutive threads: consecutive samples of a row
            const bool in = k0 + k < r;
            sa[k][row] = in ? dd_row_value(Xp, yp, m, s, lo, a0 + row, k0 + k) : 0.0;
            sb[k][row] = in ? dd_row_value(Xp, yp, m, s, lo, b0 + row, k0 + k) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < DG_K; ++k) {
            double av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                av[u] = sa[k][ty * 4 + u];
                bv[u] = sb[k][tx * 4 + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const double p = __dmul_rn(av[u], bv[v]);
                    const double e = fma(av[u], bv[v], -p);
                    const dd q = two_sum(sh[u][v], p);
                    sh[u][v] = q.hi;
                    cl[u][v] = __dadd_rn(cl[u][v], __dadd_rn(q.lo, e));
                }
        }
    }
    double* Ht = Hhi + (int64_t)t * LD * LD;
    double* Lt = Hlo + (int64_t)t * LD * LD;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t a = a0 + ty * 4 + u, b = b0 + tx * 4 + v;
            const dd h = fast_two_sum(sh[u][v], cl[u][v]);
            Ht[a * LD + b] = h.hi;
            Lt[a * LD + b] = h.lo;
            Ht[b * LD + a] = h.hi;
            Lt[b * LD + a] = h.lo;
        }
}

// ---- one thread per (tuple, task): LDL^T of the (n + 2) block in double-double ----
template <int NC>
__global__ void __launch_bounds__(128) k_dd_ill(QrArgs a, const double* __restrict__ Hhi,
                                               const double* __restrict__ Hlo, int64_t LD) {
    const int64_t g = a.g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.total) return;
    const int64_t tup_i = g / a.T;
    const int task = (int)(g % a.T);
    constexpr int n = NC - 2, p = NC - 1;
    int64_t tup[NC - 2];
    unrank_lex(a.ranks[tup_i], a.m, n, a.binom, tup);
    int64_t col[NC];
#pragma unroll
    for (int k = 0; k < n; ++k) col[k] = tup[k];
    col[n] = a.m + 1;  // the intercept's column of ones
    col[p] = a.m;      // the property
    const double* Ht = Hhi + (int64_t)task * LD * LD;
    const double* Lt = Hlo + (int64_t)task * LD * LD;
    dd L[NC][NC];
    dd d[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        // row j of L D: w_k = sum_{l<k} ... computed as c_jk = H_jk - sum_{l<k} L_jl (d_l L_kl)
#pragma unroll
        for (int k = 0; k <= j; ++k) {
            const int64_t e = col[j] * LD + col[k];
            dd v{Ht[e], Lt[e]};
#pragma unroll
            for (int l = 0; l < k; ++l) v = dd_add(v, dd_neg(dd_mul(L[j][l], dd_mul(d[l], L[k][l]))));
            if (k < j) {
                L[j][k] = (d[k].hi > 0.0) ? dd_div(v, d[k]) : dd{0.0, 0.0};
            } else {
                d[j] = v;
            }
        }
    }
    const int64_t rows = a.bounds[task + 1] - a.bounds[task];
    double mx = 0.0, mn = INFINITY;
#pragma unroll
    for (int j = 0; j < p; ++j) {
        const double v = (j < rows && d[j].hi > 0.0) ? d[j].hi + d[j].lo : 0.0;
        mx = fmax(mx, v);
        mn = fmin(mn, v);
    }
    const double dp = d[p].hi + d[p].lo;
    a.ssr[g] = (rows > p) ? fmax(dp, 0.0) : 0.0;
    a.ratio[g] = (mx > 0.0) ? sqrt(mn / mx) : 0.0;
}

}  // namespace

int64_t dd_gram_ld(int64_t m) { return (m + 2 + DG_T - 1) / DG_T * DG_T; }
// doubles of the lo buffer: T x LD x LD plus the tile list
int64_t dd_gram_lo_doubles(int64_t m, int T) {
    const int64_t LD = dd_gram_ld(m), nb = LD / DG_T;
    return (int64_t)T * LD * LD + nb * (nb + 1) / 2;
}

// The double-double screen pays for its Gram when the TSQR screen would read far more:
// TSQR ~ 60 flops per row per column pair, the Gram ~ 10 flops per (pair, row) once.
bool dd_screen_pays(int64_t nill, int n, int T, int64_t m, int64_t s) {
    const double LD = (double)dd_gram_ld(m);
    const double bytes = 2.0 * 8.0 * T * LD * LD;
    if (bytes > (double)(1ull << 30)) return false;
    const double tsqr = (double)nill * (double)s * (double)((n + 2) * (n + 2)) * 6.0;
    const double gram = 0.5 * LD * LD * (double)s * 10.0 + (double)nill * T * 40.0 * (n + 2) * (n + 2) * (n + 2);
    return gram < 0.5 * tsqr;
}

void launch_dd_screen(const QrArgs& a0, int64_t count, double* Hhi, double* Hlo, bool gram_ready, cudaStream_t st,
                      int64_t* launches) {
    const int64_t LD = dd_gram_ld(a0.m);
    if (!gram_ready) {
        const int nb = (int)(LD / DG_T);
        std::vector<int2> tl;
        for (int x = 0; x < nb; ++x)
            for (int y = x; y < nb; ++y) tl.push_back(make_int2(x, y));
        // the tile list rides behind the lo buffer's T matrices (dd_gram_lo_doubles): no
        // allocation on the stream (a cudaMallocAsync / cudaFreeAsync pair here made single
        // searches intermittently ~0.7 s slower)
        static_assert(sizeof(int2) == 8, "int2 packs into one double slot");
        int2* tiles = reinterpret_cast<int2*>(Hlo + (int64_t)a0.T * LD * LD);
        cudaMemcpyAsync(tiles, tl.data(), sizeof(int2) * tl.size(), cudaMemcpyHostToDevice, st);
        k_ddgram<<<dim3((unsigned)tl.size(), (unsigned)a0.T), 256, 0, st>>>(a0.Xp, a0.yp, a0.m, a0.s, a0.bounds, LD,
                                                                             tiles, Hhi, Hlo);
        if (launches) ++*launches;
    }
    QrArgs a = a0;
    a.total = count * a.T;
    const int64_t per_launch = (int64_t)1 << 30;
    for (int64_t g0 = 0; g0 < a.total; g0 += per_launch) {
        a.g0 = g0;
        const int64_t w = std::min(per_launch, a.total - g0);
        const unsigned blocks = (unsigned)((w + 127) / 128);
        switch (a.n) {
            case 1: k_dd_ill<3><<<blocks, 128, 0, st>>>(a, Hhi, Hlo, LD); break;
            case 2: k_dd_ill<4><<<blocks, 128, 0, st>>>(a, Hhi, Hlo, LD); break;
            case 3: k_dd_ill<5><<<blocks, 128, 0, st>>>(a, Hhi, Hlo, LD); break;
            case 4: k_dd_ill<6><<<blocks, 128, 0, st>>>(a, Hhi, Hlo, LD); break;
            case 5: k_dd_ill<7><<<blocks, 128, 0, st>>>(a, Hhi, Hlo, LD); break;
            default: k_dd_ill<8><<<blocks, 128, 0, st>>>(a, Hhi, Hlo, LD); break;  // n = 6 (l0s_qr_tuples' limit)
        }
        if (launches) ++*launches;
    }
}

}  // namespace l0s
