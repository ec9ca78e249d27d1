// stage.cu -- device staging of one search problem.
//
// Replaces search._prepare (search.py:113-127) and adds the per-task
// centering / normalization that the Gram path needs.  HBM-bound: the input
// matrix is read once for the gather and the permuted copy twice (L2-resident
// per row segment) for the statistics and the normalized write.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

// rows [f0 + GR * blockIdx.y, + GR) of [f0, f1) (row m is the property); one permutation index per
// thread serves GR rows (GR independent loads in flight, the index read once)
constexpr int GR = 8;
template <typename W>
__global__ void __launch_bounds__(256) k_gather(const double* __restrict__ values, const double* __restrict__ y,
                                                const int64_t* __restrict__ perm, int64_t m, int64_t s,
                                                W* __restrict__ Xp, W* __restrict__ yp, int64_t f0, int64_t f1) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s) return;
    const int64_t src = __ldg(perm + i);
    const int64_t fa = f0 + (int64_t)GR * blockIdx.y, fb = fa + GR < f1 ? fa + GR : f1;
    double v[GR];
#pragma unroll
    for (int r = 0; r < GR; ++r) {
        const int64_t f = fa + r;
        v[r] = f < fb ? (f < m ? values[f * s + src] : y[src]) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < GR; ++r) {
        const int64_t f = fa + r;
        if (f < fb) {
            if (f < m)
                Xp[f * s + i] = (W)v[r];  // float64 -> float32 rounds to nearest (numpy astype)
            else
                yp[i] = (W)v[r];
        }
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(L0S_FULL, v, o);
    return v;
}

// The OZ_DIGITS signed 7-bit Ozaki digits of u = z 2^-e (|u| < 1), byte a = digit a: exactly
// what the iteration v = 128 u, q_a = trunc(v), u = v - q_a (every step exact) yields, i.e.
// q_a = sign(u) (floor(|u| 2^(7(a+1))) mod 128), from one truncation of t = z p2 with
// p2 = 2^(7 OZ_DIGITS - e) (an exact scaling; |t| < 2^28) and integer field extraction.
__device__ __forceinline__ unsigned oz_digits(double z, double p2) {
    const int q = __double2int_rz(z * p2);
    const unsigned au = (unsigned)(q < 0 ? -q : q);
    if constexpr (OZ_DIGITS == 4) {
        // byte a = 7-bit digit a (most significant first); negative: every byte negated mod 256
        const unsigned w = ((au >> 21) & 127u) | (((au >> 14) & 127u) << 8) | (((au >> 7) & 127u) << 16) |
                           ((au & 127u) << 24);
        return q < 0 ? __vsub4(0u, w) : w;
    } else {
        const unsigned neg = q < 0 ? 0xffu : 0u;
        unsigned w = 0u;
#pragma unroll
        for (int a = 0; a < OZ_DIGITS; ++a) {
            const unsigned d = (au >> (7 * (OZ_DIGITS - 1 - a))) & 127u;
            w |= (((d ^ neg) + (neg & 1u)) & 0xffu) << (8 * a);  // two's complement byte of -d when negative
        }
        return w;
    }
}

// pk[a] = byte a of w[0..3] (a 4 x 4 byte transpose in 8 PRMTs)
__device__ __forceinline__ void oz_transpose4(const unsigned (&w)[4], unsigned (&pk)[4]) {
    const unsigned t0 = __byte_perm(w[0], w[1], 0x5140), t1 = __byte_perm(w[0], w[1], 0x7362);
    const unsigned u0 = __byte_perm(w[2], w[3], 0x5140), u1 = __byte_perm(w[2], w[3], 0x7362);
    pk[0] = __byte_perm(t0, u0, 0x5410);
    pk[1] = __byte_perm(t0, u0, 0x7632);
    pk[2] = __byte_perm(t1, u1, 0x5410);
    pk[3] = __byte_perm(t1, u1, 0x7632);
}

// One warp per (row, task) of rows [f0, f1); row m is the property.
// With dig.Q set, the warp also writes the row's Ozaki digits for the INT8 Gram (ozaki.cu):
// e with max |z| < 2^e, and OZ_DIGITS signed 7-bit digits of z 2^-e into each digit plane.
template <typename W>
__global__ void k_normalize(const W* __restrict__ Xp, const W* __restrict__ yp, int64_t m, int64_t s,
                            const int64_t* __restrict__ bounds, const int64_t* __restrict__ zoff, int T,
                            int64_t sp, double* __restrict__ Z, double* __restrict__ qf,
                            double* __restrict__ un2, double* __restrict__ yyu, int64_t f0, int64_t f1, DigitOut dig) {
    int lane = threadIdx.x & 31;
    int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= (f1 - f0) * T) return;
    int t = (int)(wid % T);
    int64_t f = f0 + wid / T;
    int64_t lo = bounds[t], r = bounds[t + 1] - lo;
    const W* src = (f < m) ? Xp + f * s + lo : yp + lo;
    double sum = 0.0;
    for (int64_t i = lane; i < r; i += 32) sum += (double)src[i];
    sum = warp_sum(sum);
    const double mean0 = sum / (double)r;
    // the second pass refines the mean to the rounding level of the *centered* values (an
    // offset of the computed mean would leave the columns uncentered by (mu - mean), an error the
    // Gram bound does not cover for near-constant features, mean/std ratio rho >> 1) and takes
    // the centered statistics in the same pass: with c0 = x - mean0, corr = sum c0 and
    // d = corr / r, sum (c0 - d)^2 = sum c0^2 - corr d and max |c0 - d| = max(max c0 - d, d - min c0)
    double corr = 0.0, s0 = 0.0, us = 0.0, cmax = -INFINITY, cmin = INFINITY;
    for (int64_t i = lane; i < r; i += 32) {
        const double x = (double)src[i];
        const double c = x - mean0;
        corr += c;
        s0 = fma(c, c, s0);
        us = fma(x, x, us);
        cmax = fmax(cmax, c);
        cmin = fmin(cmin, c);
    }
    corr = warp_sum(corr);
    s0 = warp_sum(s0);
    us = warp_sum(us);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cmax = fmax(cmax, __shfl_xor_sync(L0S_FULL, cmax, o));
        cmin = fmin(cmin, __shfl_xor_sync(L0S_FULL, cmin, o));
    }
    const double dlt = corr / (double)r;
    const double mean = mean0 + dlt;
    const double cs = fmax(s0 - corr * dlt, 0.0);
    const double mc = fmax(cmax - dlt, dlt - cmin);
    // features: unit-norm centered rows (0/0 -> NaN for a constant feature, which the
    // reference always rejects); property: centered, not normalized.
    double scale = (f < m) ? 1.0 / sqrt(cs) : 1.0;
    double* dst = Z + f * sp + zoff[t];
    int64_t rpad = zoff[t + 1] - zoff[t];
    if (!dig.Q) {
        for (int64_t i = lane; i < rpad; i += 32) dst[i] = (i < r) ? ((double)src[i] - mean) * scale : 0.0;
    } else {
        // every written z satisfies |z| <= fl(mc * scale) (rounding is monotone) < 2^e
        const double zmax = mc * scale;
        int e = 0;
        const bool finite = zmax > 0.0 && zmax < INFINITY;
        if (finite) frexp(zmax, &e);
        const int64_t k0 = dig.koff[t], klen = dig.koff[t + 1] - k0;
        const double p2 = finite ? ldexp(1.0, 7 * OZ_DIGITS - e) : 0.0;
        for (int64_t i = lane; i < klen; i += 32) {
            const double z = (i < r) ? ((double)src[i] - mean) * scale : 0.0;
            if (dig.write_z && i < rpad) dst[i] = z;  // Z only for a DMMA fallback (INT8 Gram: digits)
            const unsigned w = oz_digits(z, p2);
#pragma unroll
            for (int a = 0; a < OZ_DIGITS; ++a)
                dig.Q[((int64_t)a * dig.R + f) * dig.KP + k0 + i] = (int8_t)((w >> (8 * a)) & 0xffu);
        }
        if (lane == 0) {
            dig.ex[(int64_t)t * dig.R + f] = e;
            if (dig.musc) {
                dig.musc[2 * ((int64_t)t * dig.R + f)] = mean;
                dig.musc[2 * ((int64_t)t * dig.R + f) + 1] = scale;
            }
        }
    }
    if (lane == 0) {
        if (f < m) {
            qf[(int64_t)t * m + f] = cs / us;
            un2[(int64_t)t * m + f] = us;
        } else {
            yyu[t] = us;
        }
    }
}

// Fused gather + normalize: one CTA per (row, task) segment, the task's samples gathered from
// the caller's order (perm) into shared memory and the task-ordered copy (one HBM read of the
// values, one write of Xp), the statistics of k_normalize from shared memory, then the Ozaki
// digits (four 7-bit planes, 4 consecutive samples per thread: 32-bit stores) and/or Z.
// Same statistics and the same rounding of every written value as k_gather + k_normalize.
#ifndef L0S_SR_THREADS
#define L0S_SR_THREADS 256
#endif
constexpr int SR_THREADS = L0S_SR_THREADS;
template <typename W>
__global__ void __launch_bounds__(SR_THREADS) k_stage_rows(const double* __restrict__ values, const double* __restrict__ y,
                                                          const int64_t* __restrict__ perm, int64_t m, int64_t s,
                                                          const int64_t* __restrict__ bounds,
                                                          const int64_t* __restrict__ zoff, int T, int64_t sp,
                                                          W* __restrict__ Xp, W* __restrict__ yp, double* __restrict__ Z,
                                                          double* __restrict__ qf, double* __restrict__ un2,
                                                          double* __restrict__ yyu, int64_t f0, DigitOut dig) {
    extern __shared__ double seg[];
    __shared__ double red[5][SR_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = (int)(blockIdx.x % T);
    const int64_t f = f0 + blockIdx.x / T;
    const int64_t lo = bounds[t], r = bounds[t + 1] - lo;
    const double* row = f < m ? values + f * s : y;
    W* dx = f < m ? Xp + f * s + lo : yp + lo;
    // gather (+ the working dtype's rounding, numpy astype) and the first sum
    // (batches of SR_B indices, then SR_B value loads in flight per thread)
    constexpr int SR_B = 16;
    double sum = 0.0;
    for (int64_t i0 = tid; i0 < r; i0 += SR_B * SR_THREADS) {
        int64_t src[SR_B];
#pragma unroll
        for (int b = 0; b < SR_B; ++b) {
            const int64_t i = i0 + (int64_t)b * SR_THREADS;
            src[b] = i < r ? __ldg(perm + lo + i) : -1;
        }
        double v[SR_B];
#pragma unroll
        for (int b = 0; b < SR_B; ++b) v[b] = src[b] >= 0 ? row[src[b]] : 0.0;
#pragma unroll
        for (int b = 0; b < SR_B; ++b) {
            const int64_t i = i0 + (int64_t)b * SR_THREADS;
            if (i < r) {
                const W w = (W)v[b];
                dx[i] = w;
                const double x = (double)w;
                seg[i] = x;
                sum += x;
            }
        }
    }
    sum = warp_sum(sum);
    if (lane == 0) red[0][warp] = sum;
    __syncthreads();
    sum = 0.0;
#pragma unroll
    for (int w = 0; w < SR_THREADS / 32; ++w) sum += red[0][w];
    const double mean0 = sum / (double)r;
    // centered statistics around mean0 (see k_normalize: the mean refined to the centered rounding)
    double corr = 0.0, s0 = 0.0, us = 0.0, cmax = -INFINITY, cmin = INFINITY;
    for (int64_t i = tid; i < r; i += SR_THREADS) {
        const double x = seg[i];
        const double c = x - mean0;
        corr += c;
        s0 = fma(c, c, s0);
        us = fma(x, x, us);
        cmax = fmax(cmax, c);
        cmin = fmin(cmin, c);
    }
    corr = warp_sum(corr);
    s0 = warp_sum(s0);
    us = warp_sum(us);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cmax = fmax(cmax, __shfl_xor_sync(L0S_FULL, cmax, o));
        cmin = fmin(cmin, __shfl_xor_sync(L0S_FULL, cmin, o));
    }
    __syncthreads();  // red[0] is read above by every thread before being reused
    if (lane == 0) {
        red[0][warp] = corr;
        red[1][warp] = s0;
        red[2][warp] = us;
        red[3][warp] = cmax;
        red[4][warp] = cmin;
    }
    __syncthreads();
    corr = s0 = us = 0.0;
    cmax = -INFINITY;
    cmin = INFINITY;
#pragma unroll
    for (int w = 0; w < SR_THREADS / 32; ++w) {
        corr += red[0][w];
        s0 += red[1][w];
        us += red[2][w];
        cmax = fmax(cmax, red[3][w]);
        cmin = fmin(cmin, red[4][w]);
    }
    const double dlt = corr / (double)r;
    const double mean = mean0 + dlt;
    const double cs = fmax(s0 - corr * dlt, 0.0);
    const double mc = fmax(cmax - dlt, dlt - cmin);
    const double scale = (f < m) ? 1.0 / sqrt(cs) : 1.0;
    double* dst = Z + f * sp + zoff[t];
    const int64_t rpad = zoff[t + 1] - zoff[t];
    if (!dig.Q || dig.write_z)
        for (int64_t i = tid; i < rpad; i += SR_THREADS) dst[i] = (i < r) ? (seg[i] - mean) * scale : 0.0;
    if (dig.Q) {
        const double zmax = mc * scale;
        int e = 0;
        const bool finite = zmax > 0.0 && zmax < INFINITY;
        if (finite) frexp(zmax, &e);
        const int64_t k0 = dig.koff[t], klen = dig.koff[t + 1] - k0;  // multiples of 64
        const double p2 = finite ? ldexp(1.0, 7 * OZ_DIGITS - e) : 0.0;
        for (int64_t i0 = 4 * (int64_t)tid; i0 < klen; i0 += 4 * SR_THREADS) {
            unsigned pk[OZ_DIGITS] = {};
            if constexpr (OZ_DIGITS == 4) {
                // the four segment values as two 16-byte loads (no bank conflicts), digits packed
                // by a byte transpose
                double z[4];
                if (i0 + 3 < r) {
                    const double2 a01 = *reinterpret_cast<const double2*>(seg + i0);
                    const double2 a23 = *reinterpret_cast<const double2*>(seg + i0 + 2);
                    z[0] = (a01.x - mean) * scale, z[1] = (a01.y - mean) * scale;
                    z[2] = (a23.x - mean) * scale, z[3] = (a23.y - mean) * scale;
                } else {
#pragma unroll
                    for (int e4 = 0; e4 < 4; ++e4) z[e4] = i0 + e4 < r ? (seg[i0 + e4] - mean) * scale : 0.0;
                }
                unsigned w[4];
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) w[e4] = oz_digits(z[e4], p2);
                oz_transpose4(w, pk);
            } else {
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) {
                    const int64_t i = i0 + e4;
                    const double z = (i < r) ? (seg[i] - mean) * scale : 0.0;
                    const unsigned w = oz_digits(z, p2);
#pragma unroll
                    for (int a = 0; a < OZ_DIGITS; ++a) pk[a] |= ((w >> (8 * a)) & 0xffu) << (8 * e4);
                }
            }
#pragma unroll
            for (int a = 0; a < OZ_DIGITS; ++a)
                *reinterpret_cast<unsigned*>(dig.Q + ((int64_t)a * dig.R + f) * dig.KP + k0 + i0) = pk[a];
        }
        if (tid == 0) {
            dig.ex[(int64_t)t * dig.R + f] = e;
            if (dig.musc) {
                dig.musc[2 * ((int64_t)t * dig.R + f)] = mean;
                dig.musc[2 * ((int64_t)t * dig.R + f) + 1] = scale;
            }
        }
    }
    if (tid == 0) {
        if (f < m) {
            qf[(int64_t)t * m + f] = cs / us;
            un2[(int64_t)t * m + f] = us;
        } else {
            yyu[t] = us;
        }
    }
}

constexpr int64_t kStageRowsMaxSmem = 96 * 1024;

bool stage_rows_fused(int64_t max_rows, const DigitOut& dig) {
    return 8 * std::max<int64_t>(max_rows, 1) <= kStageRowsMaxSmem && !(dig.Q && dig.KP % 4 != 0);
}

void launch_stage_rows(const double* values, const double* y, const int64_t* perm, int64_t m, int64_t s, int precision,
                       void* Xp, void* yp, const int64_t* bounds_d, const int64_t* zoff_d, int T, int64_t sp,
                       double* Z, double* qf, double* un2, double* yyu, int64_t f0, int64_t f1, DigitOut dig,
                       int64_t max_rows, cudaStream_t st) {
    if (f1 <= f0) return;
    const int64_t smem = 8 * std::max<int64_t>(max_rows, 1);
    if (!stage_rows_fused(max_rows, dig)) {  // segments too long: the two passes
        launch_gather(values, y, perm, m, s, precision, Xp, yp, f0, f1, st);
        launch_normalize(Xp, yp, precision, m, s, bounds_d, zoff_d, T, sp, Z, qf, un2, yyu, f0, f1, dig, st);
        return;
    }
    const unsigned blocks = (unsigned)((f1 - f0) * T);
    if (precision == 1) {
        cudaFuncSetAttribute(k_stage_rows<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStageRowsMaxSmem);
        k_stage_rows<float><<<blocks, SR_THREADS, smem, st>>>(values, y, perm, m, s, bounds_d, zoff_d, T, sp,
                                                               (float*)Xp, (float*)yp, Z, qf, un2, yyu, f0, dig);
    } else {
        cudaFuncSetAttribute(k_stage_rows<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStageRowsMaxSmem);
        k_stage_rows<double><<<blocks, SR_THREADS, smem, st>>>(values, y, perm, m, s, bounds_d, zoff_d, T, sp,
                                                                (double*)Xp, (double*)yp, Z, qf, un2, yyu, f0, dig);
    }
}

// ---------------------------------------------------------------------------
// Per-feature conditioning flags for the screened path, on the device:
//   rho[t][f] = |f| / |f_c| = q^-1/2,  dead[f]: the reference's rank rule rejects every
//   tuple holding f,  rho_cap[t] = min(32, max rho over live features),  iforce[f]: some
//   task's rho exceeds its cap (the sweep then takes the slow path for that feature).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_reduce(double v, bool is_max, double* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        double w = __shfl_xor_sync(L0S_FULL, v, o);
        v = is_max ? fmax(v, w) : fmin(v, w);
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = sh[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = is_max ? fmax(r, sh[w]) : fmin(r, sh[w]);
        sh[0] = r;
    }
    __syncthreads();
    double r = sh[0];
    __syncthreads();
    return r;
}

__global__ void k_task_umin(const double* __restrict__ un2, int64_t m, double* __restrict__ umin,
                            const double* __restrict__ yyu, double* __restrict__ ynorm) {
    __shared__ double sh[32];
    const int t = blockIdx.x;
    if (threadIdx.x == 0) ynorm[t] = sqrt(yyu[t]);
    double v = INFINITY;
    for (int64_t f = threadIdx.x; f < m; f += blockDim.x) v = fmin(v, un2[(int64_t)t * m + f]);
    v = block_reduce(v, false, sh);
    if (threadIdx.x == 0) umin[t] = v;
}

__global__ void k_feature_flags(double tol, int fp32, const double* __restrict__ qf, const double* __restrict__ umin,
                                const double* __restrict__ rows, int64_t m, int T, double* __restrict__ rho,
                                unsigned char* __restrict__ dead) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= m) return;
    bool d = false;
    for (int t = 0; t < T; ++t) {
        const double q = qf[(int64_t)t * m + f];
        const double rf = 1.0 / sqrt(q);
        rho[(int64_t)t * m + f] = (rf == rf && rf < INFINITY) ? rf : INFINITY;
        // |R_nn| <= sqrt(r q) and max|R| >= min_f |f|: certain rejection (n <= 4 rounding model)
        const double r = rows[t];
        const double gam = fp32 ? 2.0 * 8.0 * 6.0 * (kEps32 + sqrt(r + 1.0) * kEps) : 2.0 * 8.0 * sqrt(r + 1.0) * 6.0 * kEps;
        const double lim = 0.5 * tol * sqrt(umin[t] / fmax(r, 1.0)) - 4.0 * gam;
        if (lim > 0.0 && sqrt(q) < lim) d = true;
    }
    dead[f] = d ? 1 : 0;
}

__global__ void k_task_rhocap(const double* __restrict__ rho, const unsigned char* __restrict__ dead, int64_t m,
                              double* __restrict__ cap) {
    __shared__ double sh[32];
    const int t = blockIdx.x;
    double v = 1.0;
    for (int64_t f = threadIdx.x; f < m; f += blockDim.x) {
        const double r = rho[(int64_t)t * m + f];
        if (!dead[f] && r < INFINITY) v = fmax(v, r);
    }
    v = block_reduce(v, true, sh);
    if (threadIdx.x == 0) cap[t] = fmin(32.0, v);
}

__global__ void k_feature_iforce(const double* __restrict__ rho, const double* __restrict__ cap,
                                 const unsigned char* __restrict__ dead, int64_t m, int T,
                                 unsigned char* __restrict__ iforce) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= m) return;
    bool fo = false;
    if (!dead[f])
        for (int t = 0; t < T; ++t)
            if (rho[(int64_t)t * m + f] > cap[t]) fo = true;
    iforce[f] = fo ? 1 : 0;
}

// NaN the Gram row and column of every dead feature (all tasks): its tuples then never pass the screen.
__global__ void k_mark_dead_rows(double* __restrict__ G, const unsigned char* __restrict__ dead, int64_t m, int64_t mp,
                                 int T) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    const int64_t f = blockIdx.y;
    if (f >= m || !dead[f]) return;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)T * mp;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(e / mp);
        const int64_t x = e % mp;
        double* Gt = G + (int64_t)t * mp * mp;
        Gt[f * mp + x] = nan;
        Gt[x * mp + f] = nan;
    }
}

void launch_feature_flags(double tol, int fp32, const double* qf, const double* un2, const double* rows, int64_t m, int64_t mp, int T,
                          double* umin, double* rho, double* rho_cap, unsigned char* dead, unsigned char* iforce,
                          double* G, const double* yyu, double* ynorm, cudaStream_t st) {
    const unsigned fb = (unsigned)((m + 255) / 256);
    k_task_umin<<<T, 256, 0, st>>>(un2, m, umin, yyu, ynorm);
    k_feature_flags<<<fb, 256, 0, st>>>(tol, fp32, qf, umin, rows, m, T, rho, dead);
    k_task_rhocap<<<T, 256, 0, st>>>(rho, dead, m, rho_cap);
    k_feature_iforce<<<fb, 256, 0, st>>>(rho, rho_cap, dead, m, T, iforce);
    k_mark_dead_rows<<<dim3(4, (unsigned)m), 256, 0, st>>>(G, dead, m, mp, T);
}

// one thread per (model, permuted position p): sample i = perm[p] of task t (bounds)
__global__ void k_residuals(const double* __restrict__ values, const double* __restrict__ y,
                            const int64_t* __restrict__ perm, const int64_t* __restrict__ bounds, int T, int64_t s,
                            int n, const int64_t* __restrict__ tup, const double* __restrict__ coef,
                            double* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    if (p >= s) return;
    int t = 0;
    while (t + 1 < T && p >= bounds[t + 1]) ++t;
    const int64_t i = perm[p];
    const double* ct = coef + (c * T + t) * (n + 1);
    double acc = ct[n];  // np.full(len(sl), c[-1])
    for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(ct[k], values[tup[c * n + k] * s + i]));
    out[c * s + i] = __dadd_rn(y[i], -acc);
}

void launch_residuals(const double* values, const double* y, const int64_t* perm, const int64_t* bounds, int T,
                      int64_t s, int n, const int64_t* tup, const double* coef, int64_t count, double* out,
                      cudaStream_t st) {
    if (count <= 0) return;
    k_residuals<<<dim3((unsigned)((s + 255) / 256), (unsigned)count), 256, 0, st>>>(values, y, perm, bounds, T, s, n,
                                                                                      tup, coef, out);
}

void launch_gather(const double* values, const double* y, const int64_t* perm, int64_t m, int64_t s,
                   int precision, void* Xp, void* yp, int64_t f0, int64_t f1, cudaStream_t st) {
    if (f1 <= f0) return;
    dim3 grid((unsigned)((s + 255) / 256), (unsigned)((f1 - f0 + GR - 1) / GR));
    if (precision == 1)
        k_gather<float><<<grid, 256, 0, st>>>(values, y, perm, m, s, (float*)Xp, (float*)yp, f0, f1);
    else
        k_gather<double><<<grid, 256, 0, st>>>(values, y, perm, m, s, (double*)Xp, (double*)yp, f0, f1);
}

void launch_normalize(const void* Xp, const void* yp, int precision, int64_t m, int64_t s,
                      const int64_t* bounds_d, const int64_t* zoff_d, int T, int64_t sp, double* Z,
                      double* qf, double* un2, double* yyu, int64_t f0, int64_t f1, DigitOut dig, cudaStream_t st) {
    if (f1 <= f0) return;
    int64_t warps = (f1 - f0) * T;
    unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    if (precision == 1)
        k_normalize<float><<<blocks, 256, 0, st>>>((const float*)Xp, (const float*)yp, m, s, bounds_d, zoff_d, T,
                                                   sp, Z, qf, un2, yyu, f0, f1, dig);
    else
        k_normalize<double><<<blocks, 256, 0, st>>>((const double*)Xp, (const double*)yp, m, s, bounds_d, zoff_d,
                                                    T, sp, Z, qf, un2, yyu, f0, f1, dig);
}

}  // namespace l0s
