// exact.cu -- bit-exact Householder least squares on the device.
//
// Reproduces the reference's numba kernels bit for bit:
//   _solve_inplace      lsq.py:61-110
//   score_tuples        lsq.py:113-156  (per-tuple pooled score)
//   fit_tuple_kernel    lsq.py:159-192  (coefficients, per-task ssr)
// One thread owns one (tuple, task) system and runs the reference's
// sequential loops in the reference's order.  Every operation is an explicit
// round-to-nearest intrinsic (__dmul_rn, __dadd_rn, __ddiv_rn, __dsqrt_rn,
// and the float32 ones for precision="fp32"), so nvcc cannot contract a*b+c
// into an FMA: the results equal numba's, which compiles without fast-math.
// The scratch matrix is interleaved across threads ((col*ld + row)*nthr + g)
// so that the warp's lanes touch consecutive addresses at every step.
//
// This kernel is the last stage of every search (refit of the screened
// candidates), the kernel behind fit_tuple, the path for tuples the screen
// flags as ill-conditioned, and the whole search for small instances.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {


constexpr int kMaxN = 15;

struct Scr {
    int64_t ld, nthr, g;
    __device__ __forceinline__ int64_t at(int col, int64_t row) const { return ((int64_t)col * ld + row) * nthr + g; }
};

// ---- float64 working dtype ----
__device__ bool solve_f64(double* S, const Scr& I, int64_t rows, int p, double tol, double* coef, double* ssr_out) {
    double maxdiag = 0.0;
    bool ok = true;
    for (int j = 0; j < p; ++j) {
        double nrm2 = 0.0;
        for (int64_t i = j; i < rows; ++i) {
            double v = S[I.at(j, i)];
            nrm2 = __dadd_rn(nrm2, __dmul_rn(v, v));
        }
        double nrm = __dsqrt_rn(nrm2);
        if (nrm == 0.0) {
            ok = false;
            continue;
        }
        double ajj = S[I.at(j, j)];
        double alpha = (ajj >= 0) ? -nrm : nrm;
        double vj = __dsub_rn(ajj, alpha);
        double vtv = __dadd_rn(__dsub_rn(nrm2, __dmul_rn(ajj, ajj)), __dmul_rn(vj, vj));
        S[I.at(j, j)] = vj;
        for (int c = j + 1; c <= p; ++c) {
            double w = 0.0;
            for (int64_t i = j; i < rows; ++i) w = __dadd_rn(w, __dmul_rn(S[I.at(j, i)], S[I.at(c, i)]));
            double fac = __ddiv_rn(__dmul_rn(2.0, w), vtv);
            for (int64_t i = j; i < rows; ++i) {
                int64_t o = I.at(c, i);
                S[o] = __dsub_rn(S[o], __dmul_rn(fac, S[I.at(j, i)]));
            }
        }
        S[I.at(j, j)] = alpha;
        double a = fabs(alpha);
        if (a > maxdiag) maxdiag = a;
    }
    if (ok) {
        double lim = __dmul_rn(tol, maxdiag);
        for (int j = 0; j < p; ++j)
            if (fabs(S[I.at(j, j)]) < lim) ok = false;
    }
    if (!ok) {
        *ssr_out = 0.0;
        return false;
    }
    for (int j = p - 1; j >= 0; --j) {
        double acc = S[I.at(p, j)];
        for (int c = j + 1; c < p; ++c) acc = __dsub_rn(acc, __dmul_rn(S[I.at(c, j)], coef[c]));
        coef[j] = __ddiv_rn(acc, S[I.at(j, j)]);
    }
    double ssr = 0.0;
    for (int64_t i = p; i < rows; ++i) {
        double v = S[I.at(p, i)];
        ssr = __dadd_rn(ssr, __dmul_rn(v, v));
    }
    *ssr_out = ssr;
    return true;
}

// ---- float32 working dtype: numba's mixed typing (products f32, accumulators f64) ----
__device__ bool solve_f32(float* S, const Scr& I, int64_t rows, int p, double tol, float* coef, double* ssr_out) {
    double maxdiag = 0.0;
    bool ok = true;
    for (int j = 0; j < p; ++j) {
        double nrm2 = 0.0;
        for (int64_t i = j; i < rows; ++i) {
            float v = S[I.at(j, i)];
            nrm2 = __dadd_rn(nrm2, (double)__fmul_rn(v, v));
        }
        double nrm = __dsqrt_rn(nrm2);
        if (nrm == 0.0) {
            ok = false;
            continue;
        }
        float ajj = S[I.at(j, j)];
        double alpha = (ajj >= 0) ? -nrm : nrm;
        double vj = __dsub_rn((double)ajj, alpha);
        double vtv = __dadd_rn(__dsub_rn(nrm2, (double)__fmul_rn(ajj, ajj)), __dmul_rn(vj, vj));
        S[I.at(j, j)] = __double2float_rn(vj);
        for (int c = j + 1; c <= p; ++c) {
            double w = 0.0;
            for (int64_t i = j; i < rows; ++i)
                w = __dadd_rn(w, (double)__fmul_rn(S[I.at(j, i)], S[I.at(c, i)]));
            double fac = __ddiv_rn(__dmul_rn(2.0, w), vtv);
            for (int64_t i = j; i < rows; ++i) {
                int64_t o = I.at(c, i);
                S[o] = __double2float_rn(__dsub_rn((double)S[o], __dmul_rn(fac, (double)S[I.at(j, i)])));
            }
        }
        S[I.at(j, j)] = __double2float_rn(alpha);
        double a = fabs(alpha);
        if (a > maxdiag) maxdiag = a;
    }
    if (ok) {
        double lim = __dmul_rn(tol, maxdiag);
        for (int j = 0; j < p; ++j)
            if ((double)fabsf(S[I.at(j, j)]) < lim) ok = false;
    }
    if (!ok) {
        *ssr_out = 0.0;
        return false;
    }
    for (int j = p - 1; j >= 0; --j) {
        float acc = S[I.at(p, j)];
        for (int c = j + 1; c < p; ++c) acc = __fsub_rn(acc, __fmul_rn(S[I.at(c, j)], coef[c]));
        coef[j] = __fdiv_rn(acc, S[I.at(j, j)]);
    }
    double ssr = 0.0;
    for (int64_t i = p; i < rows; ++i) {
        float v = S[I.at(p, i)];
        ssr = __dadd_rn(ssr, (double)__fmul_rn(v, v));
    }
    *ssr_out = ssr;
    return true;
}

template <typename W>
__global__ void k_exact(ExactArgs a, int64_t g0, int64_t nthr, double* __restrict__ ssr_tmp,
                        int32_t* __restrict__ ok_tmp) {
    int64_t gl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gl >= nthr) return;
    int64_t g = g0 + gl;
    int64_t tup_i = g / a.T;
    int task = (int)(g % a.T);
    if (tup_i >= a.count) return;
    int n = a.n, p = n + 1;
    int64_t tup[kMaxN];
    if (a.tuples)
        for (int k = 0; k < n; ++k) tup[k] = a.tuples[tup_i * n + k];
    else
        unrank_lex(a.ranks[tup_i], a.m, n, a.binom, tup);
    int64_t lo = a.bounds[task], rows = a.bounds[task + 1] - lo;
    Scr I{a.ld, nthr, gl};
    W* S = (W*)a.scratch;
    const W* X = (const W*)a.Xp;
    const W* Y = (const W*)a.yp;
    for (int k = 0; k < n; ++k) {
        const W* src = X + tup[k] * a.s + lo;
        for (int64_t i = 0; i < rows; ++i) S[I.at(k, i)] = src[i];
    }
    for (int64_t i = 0; i < rows; ++i) {
        S[I.at(n, i)] = (W)1.0;
        S[I.at(p, i)] = Y[lo + i];
    }
    W coef[kMaxN + 1];
    double ssr;
    bool ok;
    if constexpr (sizeof(W) == 8)
        ok = solve_f64((double*)S, I, rows, p, a.tol, (double*)coef, &ssr);
    else
        ok = solve_f32((float*)S, I, rows, p, a.tol, (float*)coef, &ssr);
    ssr_tmp[g] = ssr;
    ok_tmp[g] = ok ? 1 : 0;
    if (a.coef && ok)
        for (int k = 0; k < p; ++k) a.coef[(tup_i * a.T + task) * p + k] = (double)coef[k];
}

// ---------------------------------------------------------------------------
// Shared-memory variant: one CTA per (tuple, task) system.  The reference's
// sequential reductions stay sequential (one thread each, products and sums
// in the reference's order), but the independent ones run concurrently on
// different lanes -- the p-j dot products of step j -- and the reflection
// updates are spread over all threads.  The system lives in shared memory,
// so each sequential chain is bound by DADD latency instead of L2 latency.
// ---------------------------------------------------------------------------
template <typename W>
struct Ops;
template <>
struct Ops<double> {
    // one term of a sum of products: acc + fl(a*b)
    static __device__ __forceinline__ double term(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
    static __device__ __forceinline__ double upd(double x, double fac, double v) {
        return __dsub_rn(x, __dmul_rn(fac, v));
    }
    static __device__ __forceinline__ double widen(double x) { return x; }
    static __device__ __forceinline__ double store(double x) { return x; }
};
template <>
struct Ops<float> {
    static __device__ __forceinline__ double term(double acc, float a, float b) {
        return __dadd_rn(acc, (double)__fmul_rn(a, b));
    }
    static __device__ __forceinline__ float upd(float x, double fac, float v) {
        return __double2float_rn(__dsub_rn((double)x, __dmul_rn(fac, (double)v)));
    }
    static __device__ __forceinline__ double widen(float x) { return (double)x; }
    static __device__ __forceinline__ float store(double x) { return __double2float_rn(x); }
};

// sequential sum_{i=from}^{to-1} fl(x_i*y_i) in index order.  The loads of the next batch
// are issued before the current batch's adds, so the chain runs at DADD latency.
// B = elements per batch: 8 from shared memory, 32 from global memory (L2 latency).
template <typename W, int B = 8>
__device__ __forceinline__ double seq_dot(const W* __restrict__ x, const W* __restrict__ y, int from, int to) {
    double acc = 0.0;
    int i = from;
    if (i + B <= to) {
        W px[B], py[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            px[u] = x[i + u];
            py[u] = y[i + u];
        }
        for (; i + 2 * B <= to; i += B) {
            W nx[B], ny[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                nx[u] = x[i + B + u];
                ny[u] = y[i + B + u];
            }
#pragma unroll
            for (int u = 0; u < B; ++u) acc = Ops<W>::term(acc, px[u], py[u]);
#pragma unroll
            for (int u = 0; u < B; ++u) {
                px[u] = nx[u];
                py[u] = ny[u];
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) acc = Ops<W>::term(acc, px[u], py[u]);
        i += B;
    }
    for (; i < to; ++i) acc = Ops<W>::term(acc, x[i], y[i]);
    return acc;
}

template <typename W>
__device__ __forceinline__ void cp_async_w(W* dst, const W* src) {
    unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    if constexpr (sizeof(W) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}

// GM: the system lives in a global scratch slot (L2-resident; systems above the shared-memory
// budget) instead of shared memory; the sequential chains then prefetch 2 x 32 elements ahead.
template <typename W, bool GM = false>
__global__ void __launch_bounds__(128) k_exact_smem(ExactArgs a, int64_t g0, double* __restrict__ ssr_tmp,
                                                    int32_t* __restrict__ ok_tmp) {
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int CB = GM ? 32 : 8;  // chain prefetch batch
    W* S = GM ? reinterpret_cast<W*>(a.scratch) + (int64_t)blockIdx.x * (a.n + 2) * a.ld
              : reinterpret_cast<W*>(smraw);
    __shared__ double s_fac[kMaxN + 2];
    __shared__ double s_vtv, s_alpha;
    __shared__ int s_skip;
    __shared__ int64_t s_tup[kMaxN];
    const int tid = threadIdx.x;
    const int64_t g = g0 + blockIdx.x;
    const int64_t tup_i = g / a.T;
    const int task = (int)(g % a.T);
    const int n = a.n, p = n + 1;
    if (tid == 0) {
        if (a.tuples)
            for (int k = 0; k < n; ++k) s_tup[k] = a.tuples[tup_i * n + k];
        else
            unrank_lex(a.ranks[tup_i], a.m, n, a.binom, s_tup);
    }
    __syncthreads();
    const int64_t lo = a.bounds[task];
    const int rows = (int)(a.bounds[task + 1] - lo);
    const int ld = rows;
    const W* X = (const W*)a.Xp;
    const W* Y = (const W*)a.yp;
    // the system [f_1 .. f_n | 1 | y] (lsq.py:141-147), every element in flight at once
    if constexpr (GM) {
        for (int k = 0; k < n; ++k) {
            const W* src = X + s_tup[k] * a.s + lo;
            for (int i = tid; i < rows; i += blockDim.x) S[k * ld + i] = src[i];
        }
        for (int i = tid; i < rows; i += blockDim.x) {
            S[n * ld + i] = (W)1.0;
            S[p * ld + i] = Y[lo + i];
        }
        __threadfence_block();
    } else {
        for (int k = 0; k < n; ++k) {
            const W* src = X + s_tup[k] * a.s + lo;
            for (int i = tid; i < rows; i += blockDim.x) cp_async_w<W>(S + k * ld + i, src + i);
        }
        for (int i = tid; i < rows; i += blockDim.x) {
            S[n * ld + i] = (W)1.0;
            cp_async_w<W>(S + p * ld + i, Y + lo + i);
        }
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    double maxdiag = 0.0;  // meaningful in thread 0
    double nrm2 = 0.0;     // thread 0: norm^2 of the next column, when produced by the fused pass
    double ssr = 0.0;      // thread 0: the fused final sum of squares
    bool have = false, ok = true;
    for (int j = 0; j < p; ++j) {
        W* cj = S + j * ld;
        if (tid == 0) {
            if (!have) nrm2 = seq_dot<W, CB>(cj, cj, j, rows);
            have = false;
            double nrm = __dsqrt_rn(nrm2);
            if (nrm == 0.0) {
                ok = false;
                s_skip = 1;
            } else {
                W ajj = cj[j];
                double alpha = (ajj >= 0) ? -nrm : nrm;
                double vj = __dsub_rn(Ops<W>::widen(ajj), alpha);
                double sq = (sizeof(W) == 8) ? __dmul_rn(Ops<W>::widen(ajj), Ops<W>::widen(ajj))
                                             : (double)__fmul_rn((float)ajj, (float)ajj);
                s_vtv = __dadd_rn(__dsub_rn(nrm2, sq), __dmul_rn(vj, vj));
                s_alpha = alpha;
                cj[j] = Ops<W>::store(vj);
                s_skip = 0;
            }
        }
        __syncthreads();
        const int skip = s_skip;
        __syncthreads();  // every thread has read s_skip before thread 0 may rewrite it
        if (skip) continue;
        // w_c for c = j+1..p: independent sequential chains on lanes 0..p-j-1
        if (tid < p - j) {
            int c = j + 1 + tid;
            double w = seq_dot<W, CB>(cj, S + c * ld, j, rows);
            s_fac[c] = __ddiv_rn(__dmul_rn(2.0, w), s_vtv);
        }
        __syncthreads();
        {
            // column j+1 first, on every thread; then its sequential sum of squares (the next
            // norm, or the ssr when j+1 == p) on thread 0 while the other warps update the rest
            W* c1 = S + (j + 1) * ld;
            const double fac = s_fac[j + 1];
            for (int i = j + tid; i < rows; i += blockDim.x) c1[i] = Ops<W>::upd(c1[i], fac, cj[i]);
        }
        __syncthreads();
        if (tid == 0) {
            W* c1 = S + (j + 1) * ld;
            if (j + 1 < p) {
                nrm2 = seq_dot<W, CB>(c1, c1, j + 1, rows);
                have = true;
            } else {
                ssr = seq_dot<W, CB>(c1, c1, p, rows);
            }
        } else if (tid >= 32) {
            for (int c = j + 2; c <= p; ++c) {
                const double fac = s_fac[c];
                W* cc = S + c * ld;
                for (int i = j + tid - 32; i < rows; i += blockDim.x - 32) cc[i] = Ops<W>::upd(cc[i], fac, cj[i]);
            }
        }
        __syncthreads();
        if (tid == 0) {
            cj[j] = Ops<W>::store(s_alpha);
            double aa = fabs(s_alpha);
            if (aa > maxdiag) maxdiag = aa;
        }
    }
    if (tid != 0) return;
    if (ok) {
        double lim = __dmul_rn(a.tol, maxdiag);
        for (int j = 0; j < p; ++j)
            if (fabs(Ops<W>::widen(S[j * ld + j])) < lim) ok = false;
    }
    if (ok) {
        W coef[kMaxN + 1];
        for (int j = p - 1; j >= 0; --j) {
            W acc = S[p * ld + j];
            for (int c = j + 1; c < p; ++c) {
                if constexpr (sizeof(W) == 8)
                    acc = __dsub_rn(acc, __dmul_rn(S[c * ld + j], coef[c]));
                else
                    acc = __fsub_rn(acc, __fmul_rn(S[c * ld + j], coef[c]));
            }
            if constexpr (sizeof(W) == 8)
                coef[j] = __ddiv_rn(acc, S[j * ld + j]);
            else
                coef[j] = __fdiv_rn(acc, S[j * ld + j]);
        }
        if (a.coef)
            for (int k = 0; k < p; ++k) a.coef[(tup_i * a.T + task) * p + k] = (double)coef[k];
    } else {
        ssr = 0.0;
    }
    ssr_tmp[g] = ssr;
    ok_tmp[g] = ok ? 1 : 0;
}

// score_tuples: sum the tasks in order, stop at the first deficient one (lsq.py:148-156)
__global__ void k_exact_finalize(ExactArgs a, const double* __restrict__ ssr_tmp, const int32_t* __restrict__ ok_tmp,
                                 int64_t c0, int64_t c1) {
    int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= c1) return;
    double total = 0.0;
    bool ok = true;
    for (int t = 0; t < a.T; ++t) {
        int64_t g = c * a.T + t;
        if (!ok_tmp[g]) {
            ok = false;
            break;
        }
        total = __dadd_rn(total, ssr_tmp[g]);
    }
    if (a.ok) a.ok[c] = ok ? 1 : 0;
    if (a.score) a.score[c] = ok ? __ddiv_rn(total, (double)a.s) : __longlong_as_double(0x7ff0000000000000ll);
    if (a.ssr)
        for (int t = 0; t < a.T; ++t) a.ssr[c * a.T + t] = ok_tmp[c * a.T + t] ? ssr_tmp[c * a.T + t] : 0.0;
}

}  // namespace

void launch_exact(const ExactArgs& a, double* ssr_tmp, int32_t* ok_tmp, cudaStream_t st, int64_t* launches) {
    // ssr_tmp / ok_tmp hold count*T entries; scratch holds scratch_threads systems
    int64_t total = a.count * a.T;
    const size_t wsz = a.precision == 1 ? 4 : 8;
    const size_t smem = (size_t)a.ld * (size_t)(a.n + 2) * wsz;
    if (smem <= (size_t)200 * 1024 && a.n <= kMaxN) {
        // per device (a process may drive several, api.cu l0s_group_*): set on every call
        cudaFuncSetAttribute(k_exact_smem<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_exact_smem<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const int64_t max_grid = (int64_t)1 << 30;
        for (int64_t g0 = 0; g0 < total; g0 += max_grid) {
            unsigned blocks = (unsigned)std::min(max_grid, total - g0);
            if (a.precision == 1)
                k_exact_smem<float><<<blocks, 128, smem, st>>>(a, g0, ssr_tmp, ok_tmp);
            else
                k_exact_smem<double><<<blocks, 128, smem, st>>>(a, g0, ssr_tmp, ok_tmp);
            if (launches) ++*launches;
        }
        total = 0;  // done
    }
    if (total > 0 && total <= 8192 && a.n <= kMaxN) {
        // few large systems (the screened path's candidates): one CTA per system on an
        // L2-resident global scratch slot, scratch_threads slots per launch
        const int64_t per = std::max<int64_t>(1, a.scratch_threads);
        for (int64_t g0 = 0; g0 < total; g0 += per) {
            unsigned blocks = (unsigned)std::min(per, total - g0);
            if (a.precision == 1)
                k_exact_smem<float, true><<<blocks, 128, 0, st>>>(a, g0, ssr_tmp, ok_tmp);
            else
                k_exact_smem<double, true><<<blocks, 128, 0, st>>>(a, g0, ssr_tmp, ok_tmp);
            if (launches) ++*launches;
        }
        total = 0;
    }
    int64_t chunk = std::max<int64_t>(a.T, (a.scratch_threads / a.T) * a.T);
    for (int64_t g0 = 0; g0 < total; g0 += chunk) {
        int64_t nthr = std::min(chunk, total - g0);
        unsigned blocks = (unsigned)((nthr + 127) / 128);
        if (a.precision == 1)
            k_exact<float><<<blocks, 128, 0, st>>>(a, g0, nthr, ssr_tmp, ok_tmp);
        else
            k_exact<double><<<blocks, 128, 0, st>>>(a, g0, nthr, ssr_tmp, ok_tmp);
        if (launches) ++*launches;
    }
    if (a.count > 0) {
        k_exact_finalize<<<(unsigned)((a.count + 255) / 256), 256, 0, st>>>(a, ssr_tmp, ok_tmp, 0, a.count);
        if (launches) ++*launches;
    }
}

}  // namespace l0s
