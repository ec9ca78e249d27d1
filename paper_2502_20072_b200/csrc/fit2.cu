// fit2.cu -- screened exhaustive fit of every 2-tuple (i < j), fp64.
//
// The dimension-2 member of the screened family (fit3.cu, fit4.cu), for the
// reference's score_tuples (lsq.py:113-156) at n = 2.  Column order [j, i] of
// the centered, unit-norm features:
//   hoisted per j and task:  base = |y_c|^2 - c_j^2
//   per (i, j) and task:     g0 = C_ij,  d = 1 - g0^2,  w = c_i - g0 c_j,
//                            ssr_t = base - w^2 / d
// with the bound and certificates of fitcommon.cuh (n = 2; the hoisted 1x1 block has
// trace 1).  C(m, 2) is small next to the n = 3 and 4 spaces, so the sweep reads the Gram
// straight from L2 (coalesced C[i, j-block] rows); the selection machinery -- warp top-K'
// lists, global bound histogram, seeded threshold, slow path -- is the shared one.
//
// Unit = 32 j (lanes) x up to 1024 i, the 8 warps of a CTA taking every 8th row.
#include <algorithm>
#include <vector>

#include "fitcommon.cuh"

namespace l0s {

using namespace fit;

namespace {

constexpr int ICH2 = 1024;  // i rows per unit

// Exact lower (and optional upper) bound + certificates of one pair (i < j); see eval_tuple3.
__device__ __noinline__ int eval_tuple2(const FitArgs& a, int64_t i, int64_t j, double* lb_out,
                                        double* ub_out = nullptr) {
    const int64_t m = a.m, mp = a.mp;
    double lb = 0.0, ub = 0.0;
    bool cond = true, rank_ok = true;
    for (int t = 0; t < a.T; ++t) {
        const double* Gt = a.G + (int64_t)t * mp * mp;
        const double Y2 = Gt[m * mp + m];
        const double w0 = Gt[m * mp + j];
        const double base = Y2 - w0 * w0;
        const double trh = 1.0;
        const double* rt_ = a.rho + (int64_t)t * m;
        const double rx = fmax(rt_[i], rt_[j]);
        double At, Bt, vk;
        task_bound(2, a.eta[t], ref_gamma(a.rowsd[t], 2, a.ref_fp32), rx, Y2, a.ynorm[t], trh, At, Bt, vk);
        const double g0 = Gt[i * mp + j], ci = Gt[i * mp + m];
        const double d = fma(-g0, g0, 1.0);
        const double w = fma(-g0, w0, ci);
        const double tr = trh + (1.0 + trh) / d;
        if (!(d > 0.0) || !(vk * (1.0 + 2.0 * tr) <= FO_LIM) || !(At + Bt / d <= (a.ref_fp32 ? LOOSE32 : LOOSE) * Y2)) cond = false;
        lb += base - At - fma(w, w, Bt) / d;
        ub += base + At - fma(w, w, -Bt) / d;
        const int64_t f[2] = {i, j};
        if (!rank_certain<2>(a, t, f, tr)) rank_ok = false;
    }
    *lb_out = lb;
    if (ub_out) *ub_out = ub;
    return (cond ? 1 : 0) | (rank_ok ? 2 : 0);
}

template <int NT>
__global__ void __launch_bounds__(256, 2) k_fit2(const __grid_constant__ FitArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_unit;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m = a.m, mp = a.mp;
    const double shrink = (NT == 1) ? 1.0 : (1.0 - 2.0 * kRcpRel);
    WarpCands wc{sm + warp * CAP, reinterpret_cast<int64_t*>(sm + NW * CAP) + warp * CAP, 0,
                 a.collect == 1 ? a.theta0 : ord_dec(*(volatile unsigned long long*)a.theta_g), 0};
    const int64_t* B2 = a.binom + 2 * (m + 1);
    for (;;) {
        if (tid == 0) s_unit = atomicAdd(a.unit_counter, 1);
        __syncthreads();
        const int u = s_unit;
        __syncthreads();
        if (u >= a.n_units) break;
        const int4 U = a.units[u];
        const int j = U.x * 32 + lane;
        const int jj = j < m ? j : (int)m - 1;
        const int i_lo = U.z, i_hi = U.w;
        if (a.collect != 1) {
            const double th = fmin(hist_theta(a, lane), ord_dec(*(volatile unsigned long long*)a.theta_g));
            if (th < wc.theta) {
                wc.theta = th;
                if (lane == 0) atomicMin(a.theta_g, ord_enc(th));
            }
        }
        // hoist on j: c_j per task, K = sum_t (base_t - A_t), Bm = max_t B_t
        double w0[NT], K = 0.0, Bm = 0.0;
        bool bad = false, isnan_ = false;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const double* Gt = a.G + (int64_t)t * mp * mp;
            const double Y2 = Gt[m * mp + m];
            w0[t] = Gt[m * mp + jj];
            const double base = Y2 - w0[t] * w0[t];
            double At, Bt, vk;
            const double rh = fmax(a.rho_cap[t], a.rho[(int64_t)t * m + jj]);
            task_bound(2, a.eta[t], ref_gamma(a.rowsd[t], 2, a.ref_fp32), rh, Y2, a.ynorm[t], 1.0, At, Bt, vk);
            K += base - At;
            Bm = fmax(Bm, Bt);
            if (!(vk * 3.0 <= FO_LIM)) bad = true;
            if (w0[t] != w0[t]) isnan_ = true;
        }
        const bool valid = j < m && !isnan_;
        bool forced = false;
        double Kq = 0.0;
        auto set_kq = [&]() {
            const double x = K - wc.theta;
            forced = bad || !(x > 0.0);
            Kq = (NT == 1) ? x : x * shrink;
        };
        set_kq();
        // rows i_lo + warp + 8 r; 32 consecutive r per pending word
        for (int r0 = 0; i_lo + warp + 8 * r0 < i_hi; r0 += 32) {
            unsigned word = 0u;
#pragma unroll 4
            for (int r = 0; r < 32; ++r) {
                const int i = i_lo + warp + 8 * (r0 + r);
                const int ic = i < m ? i : (int)m - 1;
                double acc = Kq;
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const double* Gi = a.G + (int64_t)t * mp * mp + (int64_t)ic * mp;
                    const double g0 = Gi[j];
                    const double D = fma(-g0, g0, 1.0);
                    const double V = fma(-g0, w0[t], Gi[m]);
                    const double q = fma(V, V, Bm);
                    if (NT == 1)
                        acc = fma(acc, D, -q);  // (K - theta) d - q; d <= 0 also passes
                    else
                        acc = fma(-q, fabs(rcp_sweep(D)), acc);
                }
                // rho_i above rho_cap (iforce): the hoisted bound does not cover this row
                unsigned pass = (forced || a.iforce[ic]) ? 1u : ((unsigned)__double2hiint(acc) >> 31);
                if (!(valid && i < j && i < i_hi)) pass = 0u;
                word |= pass << r;
            }
            unsigned pend[1] = {word};
            drain_pending<1>(
                a, pend, wc, lane,
                [&](int b, double* lbv, int64_t* rkv) -> int {
                    const int i = i_lo + warp + 8 * (r0 + b);
                    *rkv = a.N_total - 1 - (B2[m - 1 - i] + (m - 1 - j));
                    if (a.ranged && (*rkv < a.rank_lo || *rkv >= a.rank_hi)) return 0;
                    if (bad) return 2;
                    return eval_tuple2(a, i, j, lbv) == 3 ? 1 : 2;
                },
                set_kq);
        }
    }
    flush_warp(a, wc, blockIdx.x * NW + warp, lane);
}

__global__ void __launch_bounds__(128) k_seed_eval2(const __grid_constant__ FitArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= *a.seed_n) return;
    double lb = 0.0, ub = INFINITY;
    const int fl = a.seed_tup[c * kSeedW] >= 0 ? eval_tuple2(a, a.seed_tup[c * kSeedW + 0], a.seed_tup[c * kSeedW + 1], &lb, &ub) : 0;
    a.seed_ub[c] = (fl == 3 && ub == ub) ? ub : INFINITY;
}

__global__ void k_screen2(const __grid_constant__ FitArgs a, const int64_t* __restrict__ tuples, int64_t count,
                          double* __restrict__ out_lb, int32_t* __restrict__ out_flags) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    double lb;
    out_flags[c] = eval_tuple2(a, tuples[2 * c], tuples[2 * c + 1], &lb);
    out_lb[c] = lb;
}

constexpr size_t kSmem2 = (size_t)NW * CAP * 16;

template <int NT>
int launch2(const FitArgs& a, int nsm, cudaStream_t st) {
    cudaFuncSetAttribute(k_fit2<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit2<NT>, 256, kSmem2);
    const int grid = nsm * (per_sm < 1 ? 1 : per_sm);
    if (a.collect != 1) seed_launch<2, 24>(k_seed_eval2, a, st);
    k_fit2<NT><<<grid, 256, kSmem2, st>>>(a);
    return grid;
}

template <int NT>
int grid2(int nsm) {
    cudaFuncSetAttribute(k_fit2<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit2<NT>, 256, kSmem2);
    return nsm * (per_sm < 1 ? 1 : per_sm);
}

}  // namespace

int fit2_launch(const FitArgs& a, int nsm, cudaStream_t st) {
    switch (a.T) {
        case 1: return launch2<1>(a, nsm, st);
        case 2: return launch2<2>(a, nsm, st);
        case 3: return launch2<3>(a, nsm, st);
        case 4: return launch2<4>(a, nsm, st);
        case 5: return launch2<5>(a, nsm, st);
        case 6: return launch2<6>(a, nsm, st);
        case 7: return launch2<7>(a, nsm, st);
        case 8: return launch2<8>(a, nsm, st);
        default: return a.T > 8 ? launch2<8>(a, nsm, st) : -1;  // T > 8: the first 8 tasks bound the sweep
    }
}

int fit2_grid(int T, int nsm) {
    switch (T) {
        case 1: return grid2<1>(nsm);
        case 2: return grid2<2>(nsm);
        case 3: return grid2<3>(nsm);
        case 4: return grid2<4>(nsm);
        case 5: return grid2<5>(nsm);
        case 6: return grid2<6>(nsm);
        case 7: return grid2<7>(nsm);
        case 8: return grid2<8>(nsm);
        default: return T > 8 ? grid2<8>(nsm) : -1;
    }
}

void launch_screen2(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st) {
    if (count > 0) k_screen2<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(a, tuples, count, out_lb, out_flags);
}

// Unit table for n = 2: (j-block of 32, -, i range), i < j < m, clipped to the rank range
// through prefix[v] = rank of the first pair whose smaller index is v.
std::vector<int4> fit2_units(int64_t m, const std::vector<int64_t>& c1_prefix, int64_t rank_lo, int64_t rank_hi) {
    std::vector<int4> units;
    const int nJ = (int)((m + 31) / 32);
    int i_first = 0, i_last = (int)m - 1;
    while (i_first < m && c1_prefix[i_first + 1] <= rank_lo) ++i_first;
    while (i_last > 0 && c1_prefix[i_last] >= rank_hi) --i_last;
    for (int jb = 0; jb < nJ; ++jb) {
        int i_end = (int)std::min<int64_t>((int64_t)jb * 32 + 31, m - 1);
        i_end = std::min(i_end, i_last + 1);
        for (int lo = i_first; lo < i_end; lo += ICH2) {
            const int hi = std::min(lo + ICH2, i_end);
            if (c1_prefix[hi] <= rank_lo || c1_prefix[lo] >= rank_hi) continue;
            units.push_back(make_int4(jb, 0, lo, hi));
        }
    }
    std::stable_sort(units.begin(), units.end(),
                     [](const int4& x, const int4& y) { return (x.w - x.z) > (y.w - y.z); });
    return units;
}

}  // namespace l0s
