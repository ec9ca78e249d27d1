// sis.cu -- SIS projection scores on the device, bit-identical to the reference's
// screening._chunk_scores (screening.py:126-155) with its fixed-shape pairwise sums
// (_pairwise_rowsum, screening.py:102-123).
//
// Per feature f, task t (slice sl, ns samples, weight w = ns / s), target r:
//   mean = tree(X) / ns,  Xc = X - mean,  num = tree(Xc * yc_r),  sxx = tree(Xc * Xc),
//   den = sqrt(sxx * sy_r),  r = |num| / den if den > 0 else 0,  acc_r += w * r,
//   score = clip(max_r acc_r, 0, 1)      (np.maximum propagates NaN, so does this)
// tree() is numpy's halving of a zero-padded power-of-two row: a balanced binary tree over
// contiguous ranges.  A warp owns one (feature, task): lane l folds the contiguous range
// [l E, (l+1) E) of the padded row with a binary-counter stack (the same tree, in order),
// then five shuffle levels pair adjacent lanes -- the same additions, so the same bits.
// Every operation is an explicit round-to-nearest intrinsic: nvcc would otherwise contract
// products into the following additions (FMA), which numpy never does.
// One CTA of 4 warps stages 4 feature rows (coalesced) in shared memory and gathers each
// task's samples through the slice indices from there.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {

constexpr int SIS_WARPS = 4;
constexpr int SIS_MAXR = 8;  // targets per launch

// Pairwise (balanced-tree) fold of a stream of values in index order: push a value, merge
// while the two top entries cover equal-size ranges (binary counter).  For a stream whose
// length is a power of two this is exactly numpy's halving tree.
struct Fold {
    double v[12];
    int n;  // values pushed so far
    __device__ __forceinline__ void init() { n = 0; }
    __device__ __forceinline__ void push(double x) {
        int k = n, top = __popc(n);  // stack depth = popcount(n)
        double cur = x;
        // merge while the lowest set bits of n say the top entry has the same size as cur
        while (k & 1) {
            cur = __dadd_rn(v[top - 1], cur);  // earlier range first; _rn: never contracted into an FMA
            --top;
            k >>= 1;
        }
        v[top] = cur;
        ++n;
    }
    __device__ __forceinline__ double result() const { return v[0]; }
};

// tree sum over the padded row (width W, power of two) of x(i) for i < ns (0 beyond)
template <typename Get>
__device__ __forceinline__ double warp_tree(int W, int ns, int lane, Get x) {
    const int E = W >= 32 ? W / 32 : 1;
    double part = 0.0;
    if (lane * E < W) {
        Fold f;
        f.init();
        for (int e = 0; e < E; ++e) {
            const int i = lane * E + e;
            f.push(i < ns ? x(i) : 0.0);
        }
        part = f.result();
    }
    for (int st = 1; st < 32 && st * E < W; st <<= 1) {
        const double o = __shfl_down_sync(L0S_FULL, part, st);
        if ((lane & (2 * st - 1)) == 0) part = __dadd_rn(part, o);
    }
    return __shfl_sync(L0S_FULL, part, 0);
}

__device__ __forceinline__ int pow2_ge(int n) {
    int w = 1;
    while (w < n) w <<= 1;
    return w;
}

// Target preparation: yc (task-gathered layout, R x s), sy (R x T), per target and task.
__global__ void k_sis_targets(const double* __restrict__ y, int R, int64_t s, const int64_t* __restrict__ perm,
                              const int64_t* __restrict__ bounds, int T, double* __restrict__ yc,
                              double* __restrict__ sy) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= R * T) return;
    const int r = wid / T, t = wid % T;
    const int64_t lo = bounds[t];
    const int ns = (int)(bounds[t + 1] - lo);
    const double* yr = y + (int64_t)r * s;
    double* ycr = yc + (int64_t)r * s + lo;
    if (ns == 0) {
        if (lane == 0) sy[r * T + t] = 0.0;
        return;
    }
    const int W = pow2_ge(ns);
    const double mean = warp_tree(W, ns, lane, [&](int i) { return yr[perm[lo + i]]; }) / (double)ns;
    for (int i = lane; i < ns; i += 32) ycr[i] = __dsub_rn(yr[perm[lo + i]], mean);
    __syncwarp();
    const double q = warp_tree(W, ns, lane, [&](int i) { const double v = ycr[i]; return __dmul_rn(v, v); });
    if (lane == 0) sy[r * T + t] = q;
}

// scores[f] for the rows of F (k x s, row-major, dataset sample order)
__global__ void __launch_bounds__(SIS_WARPS * 32) k_sis_scores(
    const double* __restrict__ F, int64_t k, int64_t s, const int64_t* __restrict__ perm,
    const int64_t* __restrict__ bounds, int T, const double* __restrict__ yc, const double* __restrict__ sy, int R,
    double* __restrict__ out) {
    extern __shared__ double srow[];  // SIS_WARPS rows of s doubles
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t f = (int64_t)blockIdx.x * SIS_WARPS + warp;
    double* row = srow + (int64_t)warp * s;
    if (f < k) {
        const double* src = F + f * s;
        for (int64_t i = lane; i < s; i += 32) row[i] = src[i];
    }
    __syncwarp();
    if (f >= k) return;
    const double total = (double)s;
    double acc[SIS_MAXR];
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int t = 0; t < T; ++t) {
        const int64_t lo = bounds[t];
        const int ns = (int)(bounds[t + 1] - lo);
        if (ns == 0) continue;
        const int W = pow2_ge(ns);
        const int64_t* pt = perm + lo;
        const double w = (double)ns / total;
        const double mean = warp_tree(W, ns, lane, [&](int i) { return row[pt[i]]; }) / (double)ns;
        const double sxx = warp_tree(W, ns, lane, [&](int i) {
            const double c = __dsub_rn(row[pt[i]], mean);
            return __dmul_rn(c, c);
        });
        for (int r = 0; r < R; ++r) {
            const double syr = sy[r * T + t];
            if (syr == 0.0) continue;  // the reference skips the task for this target
            const double* ycr = yc + (int64_t)r * s + lo;
            const double num = warp_tree(W, ns, lane, [&](int i) { return __dmul_rn(__dsub_rn(row[pt[i]], mean), ycr[i]); });
            const double den = __dsqrt_rn(__dmul_rn(sxx, syr));
            const double rr = (den > 0.0) ? __ddiv_rn(fabs(num), den) : 0.0;
            acc[r] = __dadd_rn(acc[r], __dmul_rn(w, rr));  // numpy: acc += w * r, two roundings
        }
    }
    if (lane == 0) {
        double best = 0.0;
        bool nan = false;
        for (int r = 0; r < R; ++r) {
            if (acc[r] != acc[r]) nan = true;
            best = acc[r] > best ? acc[r] : best;  // np.maximum; NaN handled below
        }
        double sc = nan ? __longlong_as_double(0x7ff8000000000000ll) : best;
        if (!nan) sc = sc < 0.0 ? 0.0 : (sc > 1.0 ? 1.0 : sc);
        out[f] = sc;
    }
}

}  // namespace

int sis_max_targets() { return SIS_MAXR; }

void launch_sis_targets(const double* y, int R, int64_t s, const int64_t* perm, const int64_t* bounds, int T,
                        double* yc, double* sy, cudaStream_t st) {
    const int warps = R * T;
    k_sis_targets<<<(warps * 32 + 255) / 256, 256, 0, st>>>(y, R, s, perm, bounds, T, yc, sy);
}

int launch_sis_scores(const double* F, int64_t k, int64_t s, const int64_t* perm, const int64_t* bounds, int T,
                      const double* yc, const double* sy, int R, double* out, cudaStream_t st) {
    const size_t smem = (size_t)SIS_WARPS * (size_t)s * sizeof(double);
    if (smem > 200 * 1024) return -1;
    cudaFuncSetAttribute(k_sis_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const unsigned blocks = (unsigned)((k + SIS_WARPS - 1) / SIS_WARPS);
    if (blocks) k_sis_scores<<<blocks, SIS_WARPS * 32, smem, st>>>(F, k, s, perm, bounds, T, yc, sy, R, out);
    return 0;
}

}  // namespace l0s
