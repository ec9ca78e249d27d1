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

// Two trees at once (the same shape), for two targets sharing the feature's loads.
template <int E, typename Get>
__device__ __forceinline__ double2 sb_tree2(int W, int ns, int lane, Get& x) {
    constexpr int SB = 32 * E;
    const int nsb = W > SB ? W / SB : 1;
    const int width = W / E < 32 ? W / E : 32;
    double t0 = 0.0, t1 = 0.0;
    for (int q = 0; q < nsb; ++q) {
        const int base = q * SB + lane * E;
        double p0 = 0.0, p1 = 0.0;
        if (lane < width) {
            double v0[E], v1[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (base + e < ns) {
                    const double2 xv = x(q, lane, e);
                    v0[e] = xv.x;
                    v1[e] = xv.y;
                } else {
                    v0[e] = 0.0;
                    v1[e] = 0.0;
                }
            }
#pragma unroll
            for (int st = 1; st < E; st <<= 1)
#pragma unroll
                for (int e = 0; e < E; e += 2 * st) {
                    v0[e] = __dadd_rn(v0[e], v0[e + st]);
                    v1[e] = __dadd_rn(v1[e], v1[e + st]);
                }
            p0 = v0[0];
            p1 = v1[0];
        }
        p0 = shfl_tree32(p0, lane, width);
        p1 = shfl_tree32(p1, lane, width);
        const double q0 = __shfl_sync(L0S_FULL, p0, 0), q1 = __shfl_sync(L0S_FULL, p1, 0);
        if (lane == q) {
            t0 = q0;
            t1 = q1;
        }
    }
    t0 = shfl_tree32(t0, lane, nsb);
    t1 = shfl_tree32(t1, lane, nsb);
    return make_double2(__shfl_sync(L0S_FULL, t0, 0), __shfl_sync(L0S_FULL, t1, 0));
}

template <typename Get>
__device__ __forceinline__ double2 lane_tree2_any(int W, int ns, int lane, Get x) {
    switch (W >= 512 ? 16 : (W >= 32 ? W / 32 : 1)) {
        case 1: return sb_tree2<1>(W, ns, lane, x);
        case 2: return sb_tree2<2>(W, ns, lane, x);
        case 4: return sb_tree2<4>(W, ns, lane, x);
        case 8: return sb_tree2<8>(W, ns, lane, x);
        default: return sb_tree2<16>(W, ns, lane, x);
    }
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
// warp takes features f = warp_global, += total_warps.  A feature row is read coalesced
// (cp.async, all in flight) and scattered into shared memory in task order, each task's
// segment laid out for the lane trees (lane stride E_t + 1).  The centered targets of this
// launch's group (targets r0 .. r0 + R - 1) sit in shared memory in the same layout, so the
// product trees read only shared memory.  accumulate: fold into out[] (np.maximum, NaN
// propagating) -- target groups of one chunk run as consecutive launches.
__global__ void k_sis_scores(const double* __restrict__ F, int64_t k, int64_t s, const int64_t* __restrict__ perm,
                             const int* __restrict__ dest, const int64_t* __restrict__ bounds,
                             const int* __restrict__ tE, const int* __restrict__ tpoff, int rowlen, int T,
                             const double* __restrict__ yc, const double* __restrict__ sy, int R, int accumulate,
                             double* __restrict__ out) {
    extern __shared__ double smem[];  // R target rows, then one row per warp (rowlen doubles each),
                                      // then the slot of each raw sample (int32)
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* ys = smem;
    double* row = smem + (int64_t)(R + warp) * rowlen;
    int* sdst = reinterpret_cast<int*>(smem + (int64_t)(R + nw) * rowlen);
    for (int64_t i = threadIdx.x; i < s; i += blockDim.x) sdst[i] = dest[i];  // dest[j]: slot of raw sample j
    __syncthreads();
    // yc is in task order: position p holds raw sample perm[p]
    for (int r = 0; r < R; ++r)
        for (int64_t p = threadIdx.x; p < s; p += blockDim.x) ys[(int64_t)r * rowlen + sdst[perm[p]]] = yc[(int64_t)r * s + p];
    __syncthreads();
    const double total = (double)s;
    for (int64_t f = (int64_t)blockIdx.x * nw + warp; f < k; f += (int64_t)gridDim.x * nw) {
        const double* src = F + f * s;
        // coalesced row read (raw sample order), scattered into the task-ordered layout
        for (int64_t j = lane; j < s; j += 32) cp_async8(row + sdst[j], src + j);
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
            const int off = tpoff[t];
            const double* xr = row + off;
            // element (super-block q, lane l, e) of the task's segment
            auto at = [&](int q, int l, int e) { return xr[(q * 32 + l) * (Et + 1) + e]; };
            const double w = (double)ns / total;
            const double mean = lane_tree_any(W, ns, lane, at) / (double)ns;
            // center in place (Xc = X - mean, the reference's one rounding): every later tree
            // reads Xc; a lane touches only its own slots
            {
                const int SBt = 32 * Et, nsb = W > SBt ? W / SBt : 1;
                for (int q = 0; q < nsb; ++q)
                    for (int e = 0; e < Et; ++e) {
                        if (q * SBt + lane * Et + e < ns) {
                            double* p = row + off + (q * 32 + lane) * (Et + 1) + e;
                            *p = __dsub_rn(*p, mean);
                        }
                    }
                __syncwarp();
            }
            const double sxx = lane_tree_any(W, ns, lane, [&](int q, int l, int e) {
                const double c = at(q, l, e);
                return __dmul_rn(c, c);
            });
            // targets in pairs: one pass over Xc feeds two product trees
            int r = 0;
            for (; r + 1 < R; r += 2) {
                const double sy0 = sy[r * T + t], sy1 = sy[(r + 1) * T + t];
                if (sy0 == 0.0 && sy1 == 0.0) continue;  // the reference skips the task for a target
                const double* y0 = ys + (int64_t)r * rowlen + off;
                const double* y1 = y0 + rowlen;
                const double2 num = lane_tree2_any(W, ns, lane, [&](int q, int l, int e) {
                    const int x = (q * 32 + l) * (Et + 1) + e;
                    const double c = xr[x];
                    return make_double2(__dmul_rn(c, y0[x]), __dmul_rn(c, y1[x]));
                });
                if (sy0 != 0.0) {
                    const double den = __dsqrt_rn(__dmul_rn(sxx, sy0));
                    const double rr = (den > 0.0) ? __ddiv_rn(fabs(num.x), den) : 0.0;
                    acc[r] = __dadd_rn(acc[r], __dmul_rn(w, rr));  // numpy: acc += w * r, two roundings
                }
                if (sy1 != 0.0) {
                    const double den = __dsqrt_rn(__dmul_rn(sxx, sy1));
                    const double rr = (den > 0.0) ? __ddiv_rn(fabs(num.y), den) : 0.0;
                    acc[r + 1] = __dadd_rn(acc[r + 1], __dmul_rn(w, rr));
                }
            }
            for (; r < R; ++r) {
                const double syr = sy[r * T + t];
                if (syr == 0.0) continue;
                const double* yr = ys + (int64_t)r * rowlen + off;
                const double num = lane_tree_any(W, ns, lane, [&](int q, int l, int e) {
                    const int x = (q * 32 + l) * (Et + 1) + e;
                    return __dmul_rn(xr[x], yr[x]);
                });
                const double den = __dsqrt_rn(__dmul_rn(sxx, syr));
                const double rr = (den > 0.0) ? __ddiv_rn(fabs(num), den) : 0.0;
                acc[r] = __dadd_rn(acc[r], __dmul_rn(w, rr));
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
            if (accumulate) {  // clip is monotone: max of clipped group maxima = clip of the max
                const double o = out[f];
                sc = (o != o || sc != sc) ? __longlong_as_double(0x7ff8000000000000ll) : (o > sc ? o : sc);
            }
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
    // shared memory: target rows of a group + one row per warp + the slot map; groups of targets
    // keep at least 8 warps per SM (one CTA per SM) and run as consecutive launches
    const size_t budget = 227 * 1024;
    const size_t rb = (size_t)rowlen * sizeof(double), mb = (size_t)s * sizeof(int);
    if (s > 8192 || mb + 2 * rb > budget) return -1;
    const int rows_fit = (int)((budget - mb) / rb);
    const int G = std::max(1, std::min(R, rows_fit - 8));  // targets per launch
    const int nw = std::max(1, std::min(16, rows_fit - G));
    const size_t smem = (size_t)(G + nw) * rb + mb;
    cudaFuncSetAttribute(k_sis_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    const int64_t need = (k + nw - 1) / nw;
    const unsigned blocks = (unsigned)std::min<int64_t>(need, (int64_t)nsm);
    if (!blocks) return 0;
    for (int r0 = 0; r0 < R; r0 += G) {
        const int g = std::min(G, R - r0);
        k_sis_scores<<<blocks, nw * 32, smem, st>>>(F, k, s, perm, dest, bounds, tE, tpoff, rowlen, T,
                                                    yc + (int64_t)r0 * s, sy + (int64_t)r0 * T, g, r0 > 0 ? 1 : 0,
                                                    out);
    }
    return 0;
}

}  // namespace l0s
