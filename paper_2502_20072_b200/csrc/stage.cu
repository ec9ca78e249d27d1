// stage.cu -- device staging of one search problem.
//
// Replaces search._prepare (search.py:113-127) and adds the per-task
// centering / normalization that the Gram path needs.  HBM-bound: the input
// matrix is read once for the gather and the permuted copy twice (L2-resident
// per row segment) for the statistics and the normalized write.
#include "common.cuh"
#include "kernels.h"

namespace l0s {

template <typename W>
__global__ void k_gather(const double* __restrict__ values, const double* __restrict__ y,
                         const int64_t* __restrict__ perm, int64_t m, int64_t s, W* __restrict__ Xp,
                         W* __restrict__ yp) {
    int64_t f = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t src = perm[i];
        if (f < m)
            Xp[f * s + i] = (W)values[f * s + src];  // float64 -> float32 rounds to nearest (numpy astype)
        else
            yp[i] = (W)y[src];
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(L0S_FULL, v, o);
    return v;
}

// One warp per (row, task); row m is the property.
template <typename W>
__global__ void k_normalize(const W* __restrict__ Xp, const W* __restrict__ yp, int64_t m, int64_t s,
                            const int64_t* __restrict__ bounds, const int64_t* __restrict__ zoff, int T,
                            int64_t sp, double* __restrict__ Z, double* __restrict__ qf,
                            double* __restrict__ un2, double* __restrict__ yyu) {
    int lane = threadIdx.x & 31;
    int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= (m + 1) * T) return;
    int t = (int)(wid % T);
    int64_t f = wid / T;
    int64_t lo = bounds[t], r = bounds[t + 1] - lo;
    const W* src = (f < m) ? Xp + f * s + lo : yp + lo;
    double sum = 0.0;
    for (int64_t i = lane; i < r; i += 32) sum += (double)src[i];
    sum = warp_sum(sum);
    double mean = sum / (double)r;
    // second pass refines the mean to the rounding level of the *centered* values: an offset
    // of the computed mean would leave the columns uncentered by (mu - mean), an error the
    // Gram bound does not cover for near-constant features (mean/std ratio rho >> 1)
    double corr = 0.0;
    for (int64_t i = lane; i < r; i += 32) corr += (double)src[i] - mean;
    mean += warp_sum(corr) / (double)r;
    double cs = 0.0, us = 0.0;
    for (int64_t i = lane; i < r; i += 32) {
        double x = (double)src[i];
        double c = x - mean;
        cs = fma(c, c, cs);
        us = fma(x, x, us);
    }
    cs = warp_sum(cs);
    us = warp_sum(us);
    // features: unit-norm centered rows (0/0 -> NaN for a constant feature, which the
    // reference always rejects); property: centered, not normalized.
    double scale = (f < m) ? 1.0 / sqrt(cs) : 1.0;
    double* dst = Z + f * sp + zoff[t];
    int64_t rpad = zoff[t + 1] - zoff[t];
    for (int64_t i = lane; i < rpad; i += 32) dst[i] = (i < r) ? ((double)src[i] - mean) * scale : 0.0;
    if (lane == 0) {
        if (f < m) {
            qf[(int64_t)t * m + f] = cs / us;
            un2[(int64_t)t * m + f] = us;
        } else {
            yyu[t] = us;
        }
    }
}

void launch_gather(const double* values, const double* y, const int64_t* perm, int64_t m, int64_t s,
                   int precision, void* Xp, void* yp, cudaStream_t st) {
    dim3 grid((unsigned)((s + 255) / 256 < 64 ? (s + 255) / 256 : 64), (unsigned)(m + 1));
    if (precision == 1)
        k_gather<float><<<grid, 256, 0, st>>>(values, y, perm, m, s, (float*)Xp, (float*)yp);
    else
        k_gather<double><<<grid, 256, 0, st>>>(values, y, perm, m, s, (double*)Xp, (double*)yp);
}

void launch_normalize(const void* Xp, const void* yp, int precision, int64_t m, int64_t s,
                      const int64_t* bounds_d, const int64_t* zoff_d, int T, int64_t sp, double* Z,
                      double* qf, double* un2, double* yyu, cudaStream_t st) {
    int64_t warps = (m + 1) * T;
    unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    if (precision == 1)
        k_normalize<float><<<blocks, 256, 0, st>>>((const float*)Xp, (const float*)yp, m, s, bounds_d, zoff_d, T,
                                                   sp, Z, qf, un2, yyu);
    else
        k_normalize<double><<<blocks, 256, 0, st>>>((const double*)Xp, (const double*)yp, m, s, bounds_d, zoff_d,
                                                    T, sp, Z, qf, un2, yyu);
}

}  // namespace l0s
