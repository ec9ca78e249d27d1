// sis.cu -- SIS projection scores on the device, bit-identical to the reference's
// screening._chunk_scores (screening.py:126-155) with its fixed-shape pairwise sums
// (_pairwise_rowsum, screening.py:102-123).
//
// Per feature f, task t (slice sl, ns samples, weight w = ns / s), target r:
//   mean = tree(X) / ns,  Xc = X - mean,  num = tree(Xc * yc_r),  sxx = tree(Xc * Xc),
//   den = sqrt(sxx * sy_r),  r = |num| / den if den > 0 else 0,  acc_r += w * r,
//   score = clip(max_r acc_r, 0, 1)      (np.maximum propagates NaN, so does this)
// tree() is numpy's halving of a zero-padded power-of-two row: a balanced binary tree over
// contiguous ranges.  A warp owns one feature; each task's samples are gathered (cp.async)
// into a shared-memory layout where lane l holds contiguous runs of E = min(16, W/32)
// samples (lane stride E + 1: conflict-free), summed by a register tree, then joined by
// shuffle levels between adjacent lanes and across 32 E-sample super-blocks -- the same
// additions as numpy, so the same bits.  Every operation is an explicit round-to-nearest
// intrinsic: nvcc would otherwise contract products into the following additions (FMA),
// which numpy never does.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {

constexpr int SIS_WARPS = 4;  // features (warps) per CTA
constexpr int SIS_MAXR = 8;  // targets per launch

// Balanced tree over the zero-padded power-of-two row x[0 .. W) (x(i) = 0 for i >= ns):
// numpy's halving.  The bottom five levels of every 32-element block are shuffle levels
// between adjacent lanes (lane l holds element 32 b + l: conflict-free, coalesced); the block
// sums go to a per-warp scratch (<= W / 32 <= 256 doubles) and are reduced the same way.
// Every addition is the tree's own (explicit _rn: never contracted into an FMA).
__device__ __forceinline__ double shfl_tree32(double v, int lane, int width) {
    for (int st = 1; st < width; st <<= 1) {
        const double o = __shfl_down_sync(L0S_FULL, v, st);
        if ((lane & (2 * st - 1)) == 0) v = __dadd_rn(v, o);
    }
    return v;  // meaningful at lane 0
}

template <typename Get>
__device__ __forceinline__ double warp_tree(int W, int ns, int lane, Get x, double* scratch) {
    if (W <= 32) {
        const double v = shfl_tree32(lane < ns ? x(lane) : 0.0, lane, W);
        return __shfl_sync(L0S_FULL, v, 0);
    }
    int nb = W / 32;
    for (int b = 0; b < nb; ++b) {
        const int i = b * 32 + lane;
        const double v = shfl_tree32(i < ns ? x(i) : 0.0, lane, 32);
        if (lane == 0) scratch[b] = v;
    }
    __syncwarp();
    while (nb > 32) {  // in place: block b's sum lands at b <= 32 b
        const int nn = nb / 32;
        for (int b = 0; b < nn; ++b) {
            const double v = shfl_tree32(scratch[b * 32 + lane], lane, 32);
            __syncwarp();
            if (lane == 0) scratch[b] = v;
            __syncwarp();
        }
        nb = nn;
    }
    const double v = shfl_tree32(lane < nb ? scratch[lane] : 0.0, lane, nb);
    __syncwarp();
    return __shfl_sync(L0S_FULL, v, 0);
}

// Same tree over a register-friendly layout.  With E = min(16, W / 32) and super-blocks of
// SB = 32 E elements: lane l owns the contiguous range [l E, (l+1) E) of every super-block
// (tree in registers), five shuffle levels join the 32 lanes of a super-block, and the
// W / SB <= 16 super-block sums are joined by a last shuffle tree.  x(q, l, e) reads element
// q SB + l E + e from a padded shared-memory layout (lane stride E + 1, odd: conflict-free).
template <int E, typename Get>
__device__ __forceinline__ double lane_regs(Get& x, int q, int lane, int base, int ns) {
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = (base + e < ns) ? x(q, lane, e) : 0.0;
#pragma unroll
    for (int st = 1; st < E; st <<= 1)
#pragma unroll
        for (int e = 0; e < E; e += 2 * st) v[e] = __dadd_rn(v[e], v[e + st]);
    return v[0];
}

template <int E, typename Get>
__device__ __forceinline__ double sb_tree(int W, int ns, int lane, Get& x) {
    constexpr int SB = 32 * E;
    const int nsb = W > SB ? W / SB : 1;
    const int width = W / E < 32 ? W / E : 32;
    double total = 0.0;
    for (int q = 0; q < nsb; ++q) {
        const int base = q * SB + lane * E;
        double part = (lane < width) ? lane_regs<E>(x, q, lane, base, ns) : 0.0;
        part = shfl_tree32(part, lane, width);
        // super-block sums, joined in a balanced tree: keep them on lanes 0..nsb-1
        const double pq = __shfl_sync(L0S_FULL, part, 0);
        if (lane == q) total = pq;
    }
    total = shfl_tree32(total, lane, nsb);
    return __shfl_sync(L0S_FULL, total, 0);
}

template <typename Get>
__device__ __forceinline__ double lane_tree_any(int W, int ns, int lane, Get x) {
    switch (W >= 512 ? 16 : (W >= 32 ? W / 32 : 1)) {
        case 1: return sb_tree<1>(W, ns, lane, x);
        case 2: return sb_tree<2>(W, ns, lane, x);
        case 4: return sb_tree<4>(W, ns, lane, x);
        case 8: return sb_tree<8>(W, ns, lane, x);
        default: return sb_tree<16>(W, ns, lane, x);
    }
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
    __shared__ double sscr[8][256];
    double* scratch = sscr[(threadIdx.x >> 5) & 7];
    const double mean = warp_tree(W, ns, lane, [&](int i) { return yr[perm[lo + i]]; }, scratch) / (double)ns;
    for (int i = lane; i < ns; i += 32) ycr[i] = __dsub_rn(yr[perm[lo + i]], mean);
    __syncwarp();
    const double q = warp_tree(W, ns, lane, [&](int i) { const double v = ycr[i]; return __dmul_rn(v, v); }, scratch);
    if (lane == 0) sy[r * T + t] = q;
}

// scores[f] for the rows of F (k x s, row-major, dataset sample order).  Persistent: each
// warp takes features f = warp_global, += total_warps.  A feature row is gathered (cp.async,
// all in flight) into shared memory in task order, each task's segment laid out for the lane
// trees (lane stride E_t + 1).
__global__ void __launch_bounds__(SIS_WARPS * 32) k_sis_scores(
    const double* __restrict__ F, int64_t k, int64_t s, const int64_t* __restrict__ perm,
    const int* __restrict__ dest, const int64_t* __restrict__ bounds, const int* __restrict__ tE,
    const int* __restrict__ tpoff, int rowlen, int T, const double* __restrict__ yc, const double* __restrict__ sy,
    int R, double* __restrict__ out) {
    extern __shared__ double srow[];  // SIS_WARPS rows of rowlen doubles, then src (int32), dest (int32)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* row = srow + (int64_t)warp * rowlen;
    int* ssrc = reinterpret_cast<int*>(srow + (int64_t)SIS_WARPS * rowlen);
    int* sdst = ssrc + s;
    for (int64_t i = threadIdx.x; i < s; i += blockDim.x) {
        ssrc[i] = (int)perm[i];
        sdst[i] = dest[i];
    }
    __syncthreads();
    const double total = (double)s;
    for (int64_t f = (int64_t)blockIdx.x * SIS_WARPS + warp; f < k; f += (int64_t)gridDim.x * SIS_WARPS) {
        const double* src = F + f * s;
        for (int64_t i = lane; i < s; i += 32) cp_async8(row + sdst[i], src + ssrc[i]);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        double acc[SIS_MAXR];
        for (int r = 0; r < R; ++r) acc[r] = 0.0;
        for (int t = 0; t < T; ++t) {
            const int64_t lo = bounds[t];
            const int ns = (int)(bounds[t + 1] - lo);
            if (ns == 0) continue;
            const int W = pow2_ge(ns);
            const int Et = tE[t];  // min(16, W / 32), >= 1
            const double* xr = row + tpoff[t];
            // element (super-block q, lane l, e) and its sample index within the task
            auto at = [&](int q, int l, int e) { return xr[(q * 32 + l) * (Et + 1) + e]; };
            const double w = (double)ns / total;
            const double mean = lane_tree_any(W, ns, lane, at) / (double)ns;
            const double sxx = lane_tree_any(W, ns, lane, [&](int q, int l, int e) {
                const double c = __dsub_rn(at(q, l, e), mean);
                return __dmul_rn(c, c);
            });
            for (int r = 0; r < R; ++r) {
                const double syr = sy[r * T + t];
                if (syr == 0.0) continue;  // the reference skips the task for this target
                const double* ycr = yc + (int64_t)r * s + lo;
                const int SBt = 32 * Et;
                const double num = lane_tree_any(W, ns, lane, [&](int q, int l, int e) {
                    return __dmul_rn(__dsub_rn(at(q, l, e), mean), ycr[q * SBt + l * Et + e]);
                });
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
        __syncwarp();  // the row buffer is reused by the next feature
    }
}

}  // namespace

int sis_max_targets() { return SIS_MAXR; }

void launch_sis_targets(const double* y, int R, int64_t s, const int64_t* perm, const int64_t* bounds, int T,
                        double* yc, double* sy, cudaStream_t st) {
    const int warps = R * T;
    k_sis_targets<<<(warps * 32 + 255) / 256, 256, 0, st>>>(y, R, s, perm, bounds, T, yc, sy);
}

int launch_sis_scores(const double* F, int64_t k, int64_t s, const int64_t* perm, const int* dest,
                      const int64_t* bounds, const int* tE, const int* tpoff, int rowlen, int T, const double* yc,
                      const double* sy, int R, double* out, int nsm, cudaStream_t st) {
    const size_t smem = (size_t)SIS_WARPS * (size_t)rowlen * sizeof(double) + 2 * (size_t)s * sizeof(int);
    if (smem > 200 * 1024 || s > 8192) return -1;
    cudaFuncSetAttribute(k_sis_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sis_scores, SIS_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t need = (k + SIS_WARPS - 1) / SIS_WARPS;
    const unsigned blocks = (unsigned)std::min<int64_t>(need, (int64_t)nsm * per_sm);
    if (blocks)
        k_sis_scores<<<blocks, SIS_WARPS * 32, smem, st>>>(F, k, s, perm, dest, bounds, tE, tpoff, rowlen, T, yc, sy,
                                                          R, out);
    return 0;
}

}  // namespace l0s
