// fit5.cu -- screened exhaustive fit of every 5-tuple (i < j < k < l < q), fp64.
//
// The dimension-5 member of the screened family (fit2/3/4.cu) for the reference's
// score_tuples (lsq.py:113-156) at n = 5, which otherwise ran every tuple through the
// bit-exact kernel (the reference takes any n with one code path, search.py:229).
// Column order of the centered, unit-norm LDL^T: [j, k, l, q, i].
//   hoisted per (j, k, l) (shared by the thread's P tuples) and per (j, k, l, q_p):
//     D1 = 1 - C_jk^2, L21 = (C_kl - C_jl C_jk) / D1, D2 = 1 - C_jl^2 - a21 L21,
//     L30 = C_jq, L31 = a31 / D1, L32 = a32 / D2, D3 = 1 - L30^2 - a31 L31 - a32 L32,
//     w_* the forward-substituted property column, base = |y_c|^2 - sum w_r^2 / D_r
//   per i and task (shared across q_p): g0 = C_ij, g1 = C_ik - L10 g0,
//     g2 = C_il - L20 g0 - L21 g1, D' = 1 - g0^2 - g1^2/D1 - g2^2/D2, V' likewise;
//   per q_p: g3 = C_iq - L30 g0 - L31 g1 - L32 g2, d = D' - g3^2/D3, w = V' - g3 s3,
//     ssr_t = base - w^2 / d
// with the rigorous bound and certificates of fitcommon.cuh (n = 5; the trace of the hoisted
// 4 x 4 inverse is bounded by tr_{r+1} <= tr_r + (1 + tr_r) / D_r).
//
// Unit = (32 j in lanes) x one (k, l) x (8 warps x P q's) x the i range below the j block;
// the unit table stores (j-block | q-block << 16, k | l << 16, i_lo, i_hi).  The i-dependent
// Gram rows are double-buffered in shared memory with cp.async, as in fit4.cu.
#include <algorithm>
#include <vector>

#include "fitcommon.cuh"

namespace l0s {

using namespace fit;

namespace {

template <int NT>
struct Cfg5 {
    static constexpr int P = (NT <= 2) ? 4 : 2;
    static constexpr int IB = (NT <= 2) ? 32 : 16;
    static constexpr int QSPAN = NW * P;
    static constexpr int TS = IB * (32 + QSPAN + 3);  // C[i, j-block] | C[i, q-span] | C[i, k] | C[i, l] | c_i
    static constexpr int BS = NT * TS;
    static constexpr size_t smem_bytes = (size_t)2 * BS * 8 + (size_t)NW * CAP_WIDE * 16 + (size_t)256 * P * 8;
};

// Hoisted LDL^T of (j, k, l, q) for one task (normalized, centered), plus the trace bound.
struct Hoist4 {
    double L10, rd1, s1, w0;        // (j, k)
    double L20, L21, rd2, s2;       // l
    double L30, L31, L32, rd3, s3;  // q
    double base, tr4, d1, d2, d3;
};
__device__ __forceinline__ Hoist4 hoist4(const double* Gt, int64_t mp, int64_t m, int64_t j, int64_t k, int64_t l,
                                         int64_t q) {
    Hoist4 h;
    const double Y2 = Gt[m * mp + m];
    h.w0 = Gt[m * mp + j];
    h.L10 = Gt[k * mp + j];
    h.d1 = fma(-h.L10, h.L10, 1.0);
    h.rd1 = rcp_newton(h.d1);
    const double w1 = fma(-h.L10, h.w0, Gt[m * mp + k]);
    h.s1 = w1 * h.rd1;
    h.L20 = Gt[l * mp + j];
    const double a21 = fma(-h.L20, h.L10, Gt[l * mp + k]);
    h.L21 = a21 * h.rd1;
    h.d2 = fma(-a21, h.L21, fma(-h.L20, h.L20, 1.0));
    h.rd2 = rcp_newton(h.d2);
    const double w2 = fma(-h.L21, w1, fma(-h.L20, h.w0, Gt[m * mp + l]));
    h.s2 = w2 * h.rd2;
    h.L30 = Gt[q * mp + j];
    const double a31 = fma(-h.L30, h.L10, Gt[q * mp + k]);
    h.L31 = a31 * h.rd1;
    const double a32 = fma(-h.L31, a21, fma(-h.L30, h.L20, Gt[q * mp + l]));
    h.L32 = a32 * h.rd2;
    h.d3 = fma(-a32, h.L32, fma(-a31, h.L31, fma(-h.L30, h.L30, 1.0)));
    h.rd3 = rcp_newton(h.d3);
    const double w3 = fma(-h.L32, w2, fma(-h.L31, w1, fma(-h.L30, h.w0, Gt[m * mp + q])));
    h.s3 = w3 * h.rd3;
    h.base = Y2 - h.w0 * h.w0 - w1 * h.s1 - w2 * h.s2 - w3 * h.s3;
    const double tr2 = 2.0 * h.rd1;
    const double tr3 = tr2 + (1.0 + tr2) * h.rd2;
    h.tr4 = tr3 + (1.0 + tr3) * h.rd3;
    return h;
}

// Exact lower bound + certificates of one 5-tuple (i < j < k < l < q); see eval_tuple3.
__device__ __noinline__ int eval_tuple5(const FitArgs& a, int64_t i, int64_t j, int64_t k, int64_t l, int64_t q,
                                        double* lb_out, double* ub_out = nullptr) {
    const int64_t m = a.m, mp = a.mp;
    double lb = 0.0, ub = 0.0;
    bool cond = true, rank_ok = true;
    for (int t = 0; t < a.T; ++t) {
        const double* Gt = a.G + (int64_t)t * mp * mp;
        const double Y2 = Gt[m * mp + m];
        const Hoist4 h = hoist4(Gt, mp, m, j, k, l, q);
        const double* rt_ = a.rho + (int64_t)t * m;
        const double rx = fmax(fmax(fmax(rt_[i], rt_[j]), fmax(rt_[k], rt_[l])), rt_[q]);
        double At, Bt, vk;
        task_bound(5, a.eta[t], ref_gamma(a.rowsd[t], 5, a.ref_fp32), rx, Y2, a.ynorm[t], h.tr4, At, Bt, vk);
        if (!(h.d1 > 0.0) || !(h.d2 > 0.0) || !(h.d3 > 0.0) || !(vk * (1.0 + 5.0 * h.tr4) <= FO_LIM)) cond = false;
        const double g0 = Gt[i * mp + j], ci = Gt[i * mp + m];
        const double D = fma(-g0, g0, 1.0);
        const double V = fma(-g0, h.w0, ci);
        const double g1 = fma(-h.L10, g0, Gt[i * mp + k]);
        const double D1 = fma(-g1 * h.rd1, g1, D);
        const double V1 = fma(-g1, h.s1, V);
        const double g2 = fma(-h.L21, g1, fma(-h.L20, g0, Gt[i * mp + l]));
        const double D2 = fma(-g2 * h.rd2, g2, D1);
        const double V2 = fma(-g2, h.s2, V1);
        const double g3 = fma(-h.L32, g2, fma(-h.L31, g1, fma(-h.L30, g0, Gt[i * mp + q])));
        const double d = fma(-g3 * h.rd3, g3, D2);
        const double w = fma(-g3, h.s3, V2);
        const double tr = h.tr4 + (1.0 + h.tr4) / d;
        if (!(d > 0.0) || !(vk * (1.0 + 5.0 * tr) <= FO_LIM) || !(At + Bt / d <= (a.ref_fp32 ? LOOSE32 : LOOSE) * Y2)) cond = false;
        lb += h.base - At - fma(w, w, Bt) / d;
        ub += h.base + At - fma(w, w, -Bt) / d;
        const int64_t f[5] = {i, j, k, l, q};
        if (!rank_certain<5>(a, t, f, tr)) rank_ok = false;
    }
    *lb_out = lb;
    if (ub_out) *ub_out = ub;
    return (cond ? 1 : 0) | (rank_ok ? 2 : 0);
}

template <int NT>
__global__ void __launch_bounds__(256, 1) k_fit5(const __grid_constant__ FitArgs a) {
    using C = Cfg5<NT>;
    constexpr int P = C::P, IB = C::IB, TS = C::TS, BS = C::BS, QSPAN = C::QSPAN;
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_unit;
    __shared__ unsigned char s_force[2][IB];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double* sKraw = sm + 2 * BS + 2 * NW * CAP_WIDE + tid * P;
    const int64_t m = a.m, mp = a.mp;
    const double shrink = (NT == 1) ? 1.0 : (1.0 - 2.0 * kRcpRel);
    WarpCands wc{sm + 2 * BS + warp * CAP_WIDE, reinterpret_cast<int64_t*>(sm + 2 * BS + NW * CAP_WIDE) + warp * CAP_WIDE, 0,
                 a.collect == 1 ? a.theta0 : ord_dec(*(volatile unsigned long long*)a.theta_g), 0, CAP_WIDE};
    const int64_t* B2 = a.binom + 2 * (m + 1);
    const int64_t* B3 = a.binom + 3 * (m + 1);
    const int64_t* B4 = a.binom + 4 * (m + 1);
    const int64_t* B5 = a.binom + 5 * (m + 1);

    auto load_tiles = [&](int buf, int ib0, int j0, int k, int l, int q0) {
        double* base = sm + buf * BS;
        if (tid < IB) s_force[buf][tid] = (ib0 + tid < m) ? a.iforce[ib0 + tid] : 0;
        constexpr int pr = 16 + QSPAN / 2 + 3;  // 16-byte pieces for j and q, then C[i,k], C[i,l] and c_i
        for (int x = tid; x < NT * IB * pr; x += 256) {
            const int t = x / (IB * pr), r = x % (IB * pr);
            const int row = r / pr, piece = r % pr;
            const double* Grow = a.G + (int64_t)t * mp * mp + (int64_t)(ib0 + row) * mp;
            double* Tt = base + t * TS;
            if (piece < 16)
                cp_async16(Tt + row * 32 + piece * 2, Grow + j0 + piece * 2);
            else if (piece < 16 + QSPAN / 2)
                cp_async16(Tt + IB * 32 + row * QSPAN + (piece - 16) * 2, Grow + q0 + (piece - 16) * 2);
            else if (piece == 16 + QSPAN / 2)
                cp_async8(Tt + IB * (32 + QSPAN) + row, Grow + k);
            else if (piece == 17 + QSPAN / 2)
                cp_async8(Tt + IB * (33 + QSPAN) + row, Grow + l);
            else
                cp_async8(Tt + IB * (34 + QSPAN) + row, Grow + m);
        }
        cp_async_commit();
    };

    for (;;) {
        if (tid == 0) s_unit = atomicAdd(a.unit_counter, 1);
        __syncthreads();
        const int u = s_unit;
        __syncthreads();
        if (u >= a.n_units) break;
        const int4 U = a.units[u];
        const int j0 = (U.x & 0xffff) * 32, q0 = (U.x >> 16) * QSPAN;
        const int k = U.y & 0xffff, l = U.y >> 16;
        const int j = j0 + lane;
        const int qbase = q0 + warp * P;
        const int i_lo = U.z, i_hi = U.w;
        load_tiles(0, i_lo, j0, k, l, q0);
        if (a.collect != 1) {
            const double th = fmin(hist_theta(a, lane), ord_dec(*(volatile unsigned long long*)a.theta_g));
            if (th < wc.theta) {
                wc.theta = th;
                if (lane == 0) atomicMin(a.theta_g, ord_enc(th));
            }
        }

        // ---------------- hoist ----------------
        double L10[NT], rd1[NT], s1[NT], w0[NT], L20[NT], L21[NT], rd2[NT], s2[NT];
        double L30[P][NT], L31[P][NT], L32[P][NT], rd3[P][NT], s3[P][NT], Kq[P], Bm[P];
        unsigned valid = 0, bad = 0, forced = 0;
        const int jj = j < m ? j : (int)m - 1;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int q = qbase + p;
            const int qq = q < m ? q : (int)m - 1;
            double kr = 0.0, bm = 0.0;
            bool isbad = false, isnan_ = false;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double* Gt = a.G + (int64_t)t * mp * mp;
                const double Y2 = Gt[m * mp + m];
                const Hoist4 h = hoist4(Gt, mp, m, jj, k, l, qq);
                double At, Bt, vk;
                const double* rt_ = a.rho + (int64_t)t * m;
                const double rh = fmax(fmax(a.rho_cap[t], rt_[jj]), fmax(fmax(rt_[k], rt_[l]), rt_[qq]));
                task_bound(5, a.eta[t], ref_gamma(a.rowsd[t], 5, a.ref_fp32), rh, Y2, a.ynorm[t], h.tr4, At, Bt, vk);
                L10[t] = h.L10;
                rd1[t] = h.rd1;
                s1[t] = h.s1;
                w0[t] = h.w0;
                L20[t] = h.L20;
                L21[t] = h.L21;
                rd2[t] = h.rd2;
                s2[t] = h.s2;
                L30[p][t] = h.L30;
                L31[p][t] = h.L31;
                L32[p][t] = h.L32;
                rd3[p][t] = h.rd3;
                s3[p][t] = h.s3;
                kr += h.base - At;
                bm = fmax(bm, Bt);
                if (!(h.d1 > 0.0) || !(h.d2 > 0.0) || !(h.d3 > 0.0) || !(vk * (1.0 + 5.0 * h.tr4) <= FO_LIM))
                    isbad = true;
                // dead features (NaN Gram rows) drop the tuple; a NaN from a near-singular hoisted
                // block (d1, d2 or d3 <= 0) is `bad` and goes to the exact kernel instead
                const double raw = h.w0 + h.L10 + h.L20 + h.L30 + Gt[l * mp + k] + Gt[(int64_t)qq * mp + k] +
                                   Gt[(int64_t)qq * mp + l] + Gt[m * mp + k] + Gt[m * mp + l] + Gt[m * mp + qq];
                if (raw != raw) isnan_ = true;
            }
            sKraw[p] = kr;
            Bm[p] = bm;
            if (j < k && k < l && l < q && q < m && !isnan_) valid |= 1u << p;
            if (isbad) bad |= 1u << p;
        }
        auto set_kq = [&]() {
            forced = bad;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double x = sKraw[p] - wc.theta;
                if (!(x > 0.0)) forced |= 1u << p;
                Kq[p] = x * shrink;
            }
        };
        set_kq();

        // ---------------- sweep i ----------------
        const int nib = (i_hi - i_lo + IB - 1) / IB;
        for (int bi = 0; bi < nib; ++bi) {
            const int buf = bi & 1;
            const int ib0 = i_lo + bi * IB;
            if (bi + 1 < nib) {
                load_tiles(buf ^ 1, ib0 + IB, j0, k, l, q0);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const double* T0 = sm + buf * BS;
            constexpr int NPW = (IB * P + 31) / 32;
            constexpr int IPW = 32 / P;
            unsigned pend[NPW];
#pragma unroll
            for (int pw = 0; pw < NPW; ++pw) {
                unsigned word = 0u;
#pragma unroll 1
                for (int iw = 0; iw < IPW; ++iw) {
                    const int ii = pw * IPW + iw;
                    const int i = ib0 + ii;
                    double acc[P];
#pragma unroll
                    for (int p = 0; p < P; ++p) acc[p] = Kq[p];
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        const double* Tt = T0 + t * TS;
                        const double g0 = Tt[ii * 32 + lane];
                        const double gkk = Tt[IB * (32 + QSPAN) + ii];
                        const double gll = Tt[IB * (33 + QSPAN) + ii];
                        const double ci = Tt[IB * (34 + QSPAN) + ii];
                        const double D = fma(-g0, g0, 1.0);
                        const double V = fma(-g0, w0[t], ci);
                        const double g1 = fma(-L10[t], g0, gkk);
                        const double D1 = fma(-g1 * rd1[t], g1, D);
                        const double V1 = fma(-g1, s1[t], V);
                        const double g2 = fma(-L21[t], g1, fma(-L20[t], g0, gll));
                        const double D2 = fma(-g2 * rd2[t], g2, D1);
                        const double V2 = fma(-g2, s2[t], V1);
                        double gq[P];
#pragma unroll
                        for (int p = 0; p < P; p += 2) {
                            const double2 v =
                                *reinterpret_cast<const double2*>(Tt + IB * 32 + ii * QSPAN + warp * P + p);
                            gq[p] = v.x;
                            gq[p + 1] = v.y;
                        }
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            const double g3 = fma(-L32[p][t], g2, fma(-L31[p][t], g1, fma(-L30[p][t], g0, gq[p])));
                            const double t3 = g3 * rd3[p][t];
                            const double w = fma(-g3, s3[p][t], V2);
                            const double d = fma(-t3, g3, D2);
                            const double qv = fma(w, w, Bm[p]);
                            if (NT == 1)
                                acc[p] = fma(acc[p], d, -qv);
                            else
                                acc[p] = fma(-qv, fabs(rcp_sweep(d)), acc[p]);
                        }
                    }
                    unsigned pass = forced;
#pragma unroll
                    for (int p = 0; p < P; ++p)
                        if (acc[p] < 0.0) pass |= 1u << p;
                    if (s_force[buf][ii]) pass |= (1u << P) - 1;
                    pass &= valid;
                    if (!(i < j && i < i_hi)) pass = 0;
                    word |= pass << (iw * P);
                }
                pend[pw] = word;
            }
            drain_pending<NPW>(
                a, pend, wc, lane,
                [&](int b, double* lbv, int64_t* rkv) -> int {
                    const int ii = b / P, p = b % P;
                    const int i = ib0 + ii, q = qbase + p;
                    *rkv = a.N_total - 1 -
                           (B5[m - 1 - i] + B4[m - 1 - j] + B3[m - 1 - k] + B2[m - 1 - l] + (m - 1 - q));
                    if (a.ranged && (*rkv < a.rank_lo || *rkv >= a.rank_hi)) return 0;
                    if ((bad >> p) & 1u) return 2;
                    return eval_tuple5(a, i, j, k, l, q, lbv) == 3 ? 1 : 2;
                },
                set_kq);
            __syncthreads();
        }
    }
    flush_warp(a, wc, blockIdx.x * NW + warp, lane);
}

__global__ void k_screen5(const __grid_constant__ FitArgs a, const int64_t* __restrict__ tuples, int64_t count,
                          double* __restrict__ out_lb, int32_t* __restrict__ out_flags) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    double lb;
    const int64_t* t = tuples + 5 * c;
    out_flags[c] = eval_tuple5(a, t[0], t[1], t[2], t[3], t[4], &lb);
    out_lb[c] = lb;
}

template <int NT>
int occupancy5(int nsm) {
    using C = Cfg5<NT>;
    cudaFuncSetAttribute(k_fit5<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit5<NT>, 256, C::smem_bytes);
    return nsm * (per_sm < 1 ? 1 : per_sm);
}

__global__ void __launch_bounds__(128) k_seed_eval5(const __grid_constant__ FitArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= *a.seed_n) return;
    double lb = 0.0, ub = INFINITY;
    const int64_t* f = a.seed_tup + (int64_t)c * kSeedW;
    const int fl = f[0] >= 0 ? eval_tuple5(a, f[0], f[1], f[2], f[3], f[4], &lb, &ub) : 0;
    a.seed_ub[c] = (fl == 3 && ub == ub) ? ub : INFINITY;
}

template <int NT>
int launch5(const FitArgs& a, int nsm, cudaStream_t st) {
    const int grid = occupancy5<NT>(nsm);
    if (a.collect != 1) seed_launch<5, 12>(k_seed_eval5, a, st);
    k_fit5<NT><<<grid, 256, Cfg5<NT>::smem_bytes, st>>>(a);
    return grid;
}

}  // namespace

void launch_screen5(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st) {
    if (count > 0) k_screen5<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(a, tuples, count, out_lb, out_flags);
}

int fit5_qspan(int T) { return T <= 2 ? Cfg5<1>::QSPAN : Cfg5<4>::QSPAN; }

// More than 4 tasks: the sweep bounds with the first 4 (every task's SSR is >= 0); the slow
// path, the certificates and the exact refit take every task.
int fit5_grid(int T, int nsm) {
    switch (T) {
        case 1: return occupancy5<1>(nsm);
        case 2: return occupancy5<2>(nsm);
        case 3: return occupancy5<3>(nsm);
        default: return T >= 4 ? occupancy5<4>(nsm) : -1;
    }
}

int fit5_launch(const FitArgs& a, int nsm, cudaStream_t st) {
    switch (a.T) {
        case 1: return launch5<1>(a, nsm, st);
        case 2: return launch5<2>(a, nsm, st);
        case 3: return launch5<3>(a, nsm, st);
        default: return a.T >= 4 ? launch5<4>(a, nsm, st) : -1;
    }
}

// Unit table for n = 5: (j-block | q-block << 16, k | l << 16, i_lo, i_hi), i < j < k < l < q < m.
// c4_prefix[v] = rank of the first tuple whose smallest index is v.
std::vector<int4> fit5_units(int64_t m, int T, const std::vector<int64_t>& c4_prefix, int64_t rank_lo,
                             int64_t rank_hi) {
    const int qspan = fit5_qspan(T);
    const int ich = 128;
    std::vector<int4> units;
    const int nJ = (int)((m + 31) / 32);
    const int nQ = (int)((m + qspan - 1) / qspan);
    int i_first = 0, i_last = (int)m - 1;
    while (i_first < m && c4_prefix[i_first + 1] <= rank_lo) ++i_first;
    while (i_last > 0 && c4_prefix[i_last] >= rank_hi) --i_last;
    for (int jb = 0; jb < nJ; ++jb) {
        const int jlo = jb * 32;
        int i_end = (int)std::min<int64_t>(jlo + 31, m - 4);
        i_end = std::min(i_end, i_last + 1);
        if (i_end <= i_first) continue;
        for (int k = jlo + 1; k <= m - 3; ++k) {
            for (int l = k + 1; l <= m - 2; ++l) {
                for (int qb = (l + 1) / qspan; qb < nQ; ++qb) {
                    if ((int64_t)qb * qspan + qspan - 1 <= l) continue;
                    for (int lo = i_first; lo < i_end; lo += ich) {
                        const int hi = std::min(lo + ich, i_end);
                        if (c4_prefix[hi] <= rank_lo || c4_prefix[lo] >= rank_hi) continue;
                        units.push_back(make_int4(jb | (qb << 16), k | (l << 16), lo, hi));
                    }
                }
            }
        }
    }
    std::stable_sort(units.begin(), units.end(),
                     [](const int4& x, const int4& y) { return (x.w - x.z) > (y.w - y.z); });
    return units;
}

}  // namespace l0s
