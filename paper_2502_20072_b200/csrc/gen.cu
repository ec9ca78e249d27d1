// gen.cu -- final-rung candidate evaluation on the device.
//
// Replaces the value half of the reference's streamed last rung
// (generation.iter_final_rung, generation.py:331-393): for a chunk of child
// pairs of one operator, each candidate's value vector
// (expressions.apply_operator_values, expressions.py:168-192), its validity
// (generation._validity_mask, generation.py:107-118) and a 128-bit fingerprint
// of the vector rounded to the dedup tolerance (the role of
// generation.value_fingerprint, generation.py:78-88: equal rounded vectors,
// equal fingerprints).  One warp per candidate, lanes striding the samples;
// the pool (rung < max) stays resident in HBM, so a candidate costs two L2
// row reads and one fp64 row write (kept for the SIS scores).
//
// Only operators whose numpy value is a single IEEE-rounded operation per
// element (or a fixed sequence of them) are evaluated here, with explicit
// _rn intrinsics so no FMA contraction changes a bit: add, sub, mul, div,
// abs_diff, sqrt, sq, cb, inv, abs.  libm operators (exp, log, sin, cos, cbrt,
// a**6) arrive as precomputed values (kind GEN_VALUES) -- a GPU libm differs
// from numpy's in the last ulp, which would move validity and dedup decisions.
#include <algorithm>
#include <cstdint>

#include "kernels.h"

namespace l0s {

namespace {

__device__ __forceinline__ double op_apply(int kind, double a, double b) {
    switch (kind) {
        case GEN_ADD: return __dadd_rn(a, b);
        case GEN_SUB: return __dsub_rn(a, b);
        case GEN_MUL: return __dmul_rn(a, b);
        case GEN_DIV: return __ddiv_rn(a, b);
        case GEN_ABS_DIFF: return fabs(__dsub_rn(a, b));
        case GEN_SQRT: return __dsqrt_rn(a);
        case GEN_SQ: return __dmul_rn(a, a);
        case GEN_CB: return __dmul_rn(__dmul_rn(a, a), a);
        case GEN_INV: return __ddiv_rn(1.0, a);
        case GEN_ABS: return fabs(a);
        default: return a;  // GEN_COPY / GEN_VALUES
    }
}

__device__ __forceinline__ float op_apply(int kind, float a, float b) {
    switch (kind) {
        case GEN_ADD: return __fadd_rn(a, b);
        case GEN_SUB: return __fsub_rn(a, b);
        case GEN_MUL: return __fmul_rn(a, b);
        case GEN_DIV: return __fdiv_rn(a, b);
        case GEN_ABS_DIFF: return fabsf(__fsub_rn(a, b));
        case GEN_SQRT: return __fsqrt_rn(a);
        case GEN_SQ: return __fmul_rn(a, a);
        case GEN_CB: return __fmul_rn(__fmul_rn(a, a), a);
        case GEN_INV: return __fdiv_rn(1.0f, a);
        case GEN_ABS: return fabsf(a);
        default: return a;
    }
}

// splitmix64 finalizer: a bijection of 64-bit words
__device__ __forceinline__ unsigned long long mix64(unsigned long long u) {
    u ^= u >> 30;
    u *= 0xbf58476d1ce4e5b9ull;
    u ^= u >> 27;
    u *= 0x94d049bb133111ebull;
    u ^= u >> 31;
    return u;
}

// T = the pool's dtype (numpy keeps the children's dtype).  A = pool rows (n_pool x s), or the
// candidates' own precomputed rows for GEN_VALUES.  Outputs: vals (count x s, fp64 -- exact for
// both dtypes), valid (count), hash (count x 2).
template <typename T>
__global__ void k_gen_eval(const T* __restrict__ A, int64_t s, const int* __restrict__ pi, const int* __restrict__ pj,
                           int count, int kind, double tol, double min_abs, double max_abs, double dedup_tol,
                           double* __restrict__ vals, unsigned char* __restrict__ valid,
                           unsigned long long* __restrict__ hash) {
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= count) return;
    const T* a = A + (int64_t)(kind == GEN_VALUES ? c : pi[c]) * s;
    const int jb = (kind == GEN_VALUES || pj == nullptr) ? -1 : pj[c];
    const T* b = jb >= 0 ? A + (int64_t)jb * s : a;
    double* out = vals ? vals + (int64_t)c * s : nullptr;
    bool finite = true;
    T amax = (T)0, vmax = (T)0, vmin = (T)0;
    bool first = true;
    unsigned long long h1 = 0, h2 = 0;
    for (int64_t e = lane; e < s; e += 32) {
        const T v = op_apply(kind, a[e], b[e]);
        if (out) out[e] = (double)v;
        finite &= isfinite(v);
        const T av = v < (T)0 ? -v : v;
        if (first) {
            amax = av;
            vmax = v;
            vmin = v;
            first = false;
        } else {
            amax = av > amax ? av : amax;
            vmax = v > vmax ? v : vmax;
            vmin = v < vmin ? v : vmin;
        }
        // the value the fingerprint sees: float64(v), rounded to the tolerance (np.round: half
        // to even), + 0.0 so that -0 and +0 agree (generation.py:85-87)
        double x = (double)v;
        if (tol > 0.0) x = rint(__ddiv_rn(x, tol));
        x = __dadd_rn(x, 0.0);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
        h1 += mix64(bits ^ ((unsigned long long)(e + 1) * 0x9e3779b97f4a7c15ull));
        h2 += mix64((bits + 0x632be59bd9b4e019ull) ^ ((unsigned long long)(e + 1) * 0xd6e8feb86659fd93ull));
    }
    // warp reductions (lanes without elements carry first = true)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        finite &= __shfl_xor_sync(0xffffffffu, (int)finite, o) != 0;
        h1 += __shfl_xor_sync(0xffffffffu, h1, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
        const T oa = __shfl_xor_sync(0xffffffffu, amax, o);
        const T ox = __shfl_xor_sync(0xffffffffu, vmax, o);
        const T on = __shfl_xor_sync(0xffffffffu, vmin, o);
        const bool of = __shfl_xor_sync(0xffffffffu, (int)first, o) != 0;
        if (!of) {
            if (first) {
                amax = oa;
                vmax = ox;
                vmin = on;
                first = false;
            } else {
                amax = oa > amax ? oa : amax;
                vmax = ox > vmax ? ox : vmax;
                vmin = on < vmin ? on : vmin;
            }
        }
    }
    if (lane == 0) {
        // _validity_mask in the pool's dtype: the Python-float limits are weak scalars (NEP 50),
        // i.e. compared after rounding to T; the spread is a T subtraction
        bool ok = finite && s > 0;
        if (ok) {
            const T spread = vmax - vmin;
            ok = amax <= (T)max_abs && amax >= (T)min_abs && spread > (T)dedup_tol;
        }
        valid[c] = ok ? 1 : 0;
        hash[2 * c] = h1;
        hash[2 * c + 1] = h2;
    }
}

// rows[i] of vals (fp64) -> out[i] in the pool's dtype (exact: the values were T)
template <typename T>
__global__ void k_gen_gather(const double* __restrict__ vals, int64_t s, const int* __restrict__ rows, int count,
                             T* __restrict__ out) {
    const int64_t n = (int64_t)count * s;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = x / s, e = x % s;
        out[x] = (T)vals[(int64_t)rows[r] * s + e];
    }
}

}  // namespace

void launch_gen_gather(const double* vals, int64_t s, const int* rows, int count, int fp32, void* out,
                       cudaStream_t st) {
    if (count <= 0 || s <= 0) return;
    const int64_t n = (int64_t)count * s;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (fp32)
        k_gen_gather<float><<<blocks, 256, 0, st>>>(vals, s, rows, count, (float*)out);
    else
        k_gen_gather<double><<<blocks, 256, 0, st>>>(vals, s, rows, count, (double*)out);
}

void launch_gen_eval(const void* A, int fp32, int64_t s, const int* pi, const int* pj, int count, int kind, double tol,
                     double min_abs, double max_abs, double dedup_tol, double* vals, unsigned char* valid,
                     unsigned long long* hash, cudaStream_t st) {
    if (count <= 0) return;
    const unsigned blocks = (unsigned)(((int64_t)count * 32 + 255) / 256);
    if (fp32)
        k_gen_eval<float><<<blocks, 256, 0, st>>>((const float*)A, s, pi, pj, count, kind, tol, min_abs, max_abs,
                                                  dedup_tol, vals, valid, hash);
    else
        k_gen_eval<double><<<blocks, 256, 0, st>>>((const double*)A, s, pi, pj, count, kind, tol, min_abs, max_abs,
                                                   dedup_tol, vals, valid, hash);
}

}  // namespace l0s
