// fit4.cu -- screened exhaustive fit of every 4-tuple (i < j < k < l), fp64.
//
// Same scheme as fit3.cu with one more hoisted column.  Column order of the
// centered, unit-norm LDL^T is [j, k, l, i]:
//   hoisted per (j, k) (shared by the thread's P tuples) and per (j, k, l_p),
//   per i and task: g0 = C_ij, g1 = C_ik - C_jk g0 (shared across l_p),
//                   g2 = C_il - L20 g0 - L21 g1,
//                   d  = 1 - g0^2 - g1^2/d1 - g2^2/d2,  w = c_i - g0 c_j - g1 s1 - g2 s2,
//                   ssr_t = base - w^2/d   (7 FP64 ops per tuple-task + 6 shared per row)
// with the bound and certificates of fitcommon.cuh (n = 4).
//
// Unit = (32 j in lanes) x one k x (8 warps x P l's) x up to 128 i; the unit
// table stores (j-block | l-block << 16, k, i_lo, i_hi).
#include <algorithm>
#include <vector>

#include "fitcommon.cuh"

namespace l0s {

using namespace fit;

namespace {

template <int NT>
struct Cfg4 {
    static constexpr int P = (NT <= 2) ? 4 : 2;
    static constexpr int IB = (NT <= 2) ? 32 : 16;
    static constexpr int LSPAN = NW * P;
    static constexpr int TS = IB * (32 + LSPAN + 2);  // C[i, j-block] | C[i, l-span] | C[i, k] | c_i
    static constexpr int BS = NT * TS;
    static constexpr size_t smem_bytes = (size_t)2 * BS * 8 + (size_t)NW * CAP_WIDE * 16 + (size_t)256 * P * 8;
};

// Hoisted LDL^T of (j, k, l) for one task (normalized, centered), plus the bound's trace term.
struct Hoist3 {
    double L10, rd1, s1, w0;   // (j, k) part
    double L20, L21, rd2, s2;  // l part
    double base, tr3, d1, d2;
};
__device__ __forceinline__ Hoist3 hoist3(const double* Gt, int64_t mp, int64_t m, int64_t j, int64_t k, int64_t l) {
    Hoist3 h;
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
    h.base = Y2 - h.w0 * h.w0 - w1 * h.s1 - w2 * h.s2;
    const double tr2 = 2.0 * h.rd1;
    h.tr3 = tr2 + (1.0 + tr2) * h.rd2;
    return h;
}

// Exact lower bound + certificates of one 4-tuple (i < j < k < l); see eval_tuple3.
__device__ __noinline__ int eval_tuple4(const FitArgs& a, int64_t i, int64_t j, int64_t k, int64_t l,
                                        double* lb_out, double* ub_out = nullptr) {
    const int64_t m = a.m, mp = a.mp;
    double lb = 0.0, ub = 0.0;
    bool cond = true, rank_ok = true;
    for (int t = 0; t < a.T; ++t) {
        const double* Gt = a.G + (int64_t)t * mp * mp;
        const double Y2 = Gt[m * mp + m];
        const Hoist3 h = hoist3(Gt, mp, m, j, k, l);
        const double* rt_ = a.rho + (int64_t)t * m;
        const double rx = fmax(fmax(rt_[i], rt_[j]), fmax(rt_[k], rt_[l]));
        double At, Bt, vk;
        task_bound(4, a.eta[t], ref_gamma(a.rowsd[t], 4, a.ref_fp32), rx, Y2, a.ynorm[t], h.tr3, At, Bt, vk);
        if (!(h.d1 > 0.0) || !(h.d2 > 0.0) || !(vk * (1.0 + 4.0 * h.tr3) <= FO_LIM)) cond = false;
        const double g0 = Gt[i * mp + j], ci = Gt[i * mp + m];
        const double D = fma(-g0, g0, 1.0);
        const double V = fma(-g0, h.w0, ci);
        const double g1 = fma(-h.L10, g0, Gt[i * mp + k]);
        const double t1 = g1 * h.rd1;
        const double D1 = fma(-t1, g1, D);
        const double V1 = fma(-g1, h.s1, V);
        const double g2 = fma(-h.L21, g1, fma(-h.L20, g0, Gt[i * mp + l]));
        const double t2 = g2 * h.rd2;
        const double d = fma(-t2, g2, D1);
        const double w = fma(-g2, h.s2, V1);
        const double tr = h.tr3 + (1.0 + h.tr3) / d;
        if (!(d > 0.0) || !(vk * (1.0 + 4.0 * tr) <= FO_LIM) || !(At + Bt / d <= (a.ref_fp32 ? LOOSE32 : LOOSE) * Y2)) cond = false;
        lb += h.base - At - fma(w, w, Bt) / d;
        ub += h.base + At - fma(w, w, -Bt) / d;
        const int64_t f[4] = {i, j, k, l};
        if (!rank_certain<4>(a, t, f, tr)) rank_ok = false;
    }
    *lb_out = lb;
    if (ub_out) *ub_out = ub;
    return (cond ? 1 : 0) | (rank_ok ? 2 : 0);
}

// Tile screen of the n = 4 sweep (fit3.cu's TSK, one task slot t0 -- the task of largest |y_c|^2,
// whose row-block maxima k_tile_max holds): with a = max |C_ij| (j-block), b_k = max |C_ik|,
// b_l = max |C_il_p|, c = max |c_i| over an i-tile,
//   |g1| <= G1 = b_k + |L10| a,  |g2| <= G2 = b_l + |L20| a + |L21| G1,
//   d >= 1 - a^2 - G1^2 / d1 - G2^2 / d2,  |w| <= c + a |c_j| + G1 |s1| + G2 |s2|,
// and a tile is retired for the warp when (K0 - theta) d_min > (w_max^2 + Bm)(1 + 4 kRcpRel) for
// every valid, unforced pair: every tuple of it has t0's share of the pooled bound at or above
// the threshold (the pooled SSR is at least that share: every task's SSR is >= 0).  Lanes gather
// the maxima of tile `lane` (a unit holds at most 128 rows); returns this warp's need bits.
struct Slot4 {
    double la10, rd1, as1, aw0;  // |L10|, 1/d1 (1 + 2e-14), |s1|, |c_j| of slot t0
};
template <int P, int IB>
__device__ __noinline__ unsigned tile_screen4(const FitArgs& a, const Slot4 h, const double (&l20)[P],
                                              const double (&l21)[P], const double (&rd2)[P], const double (&as2)[P],
                                              const double (&kq)[P], const double (&bm)[P], unsigned valid,
                                              unsigned cand, int lane, int jb, int k, int lbase, int i_lo, int i_hi,
                                              int nib) {
    const int64_t m = a.m;
    if (__any_sync(L0S_FULL, (valid & ~cand) != 0u)) return (nib >= 32) ? ~0u : ((1u << nib) - 1u);
    const int nbk = (int)((m + IB - 1) / IB);
    const double* MT = a.tmax;
    const double* MJ = a.tmax + (m + 1) * nbk + (int64_t)jb * nbk;
    double amx = 0.0, bkx = 0.0, cmx = 0.0, blx[P];
#pragma unroll
    for (int p = 0; p < P; ++p) blx[p] = 0.0;
    if (lane < nib) {
        const int r0 = i_lo + lane * IB, r1 = min(r0 + IB, i_hi);
        for (int b = r0 / IB; b <= (r1 - 1) / IB; ++b) {
            amx = fmax(amx, MJ[b]);
            bkx = fmax(bkx, MT[(int64_t)k * nbk + b]);
            cmx = fmax(cmx, MT[m * nbk + b]);
#pragma unroll
            for (int p = 0; p < P; ++p) blx[p] = fmax(blx[p], MT[(int64_t)(lbase + p < m ? lbase + p : m - 1) * nbk + b]);
        }
    }
    unsigned word = 0u;
    for (int bb = 0; bb < nib; ++bb) {
        const double am = __shfl_sync(L0S_FULL, amx, bb), bk = __shfl_sync(L0S_FULL, bkx, bb);
        const double cm = __shfl_sync(L0S_FULL, cmx, bb);
        const double G1 = fma(h.la10, am, bk) * (1.0 + 1e-15);
        const double c1 = fma(-G1 * G1, h.rd1, fma(-am, am, 1.0 - 1e-14));
        const double w1 = fma(G1, h.as1, fma(am, h.aw0, cm));
        bool need = false;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const double bl = __shfl_sync(L0S_FULL, blx[p], bb);
            if (!((valid >> p) & 1u)) continue;
            const double G2 = fma(fabs(l21[p]), G1, fma(fabs(l20[p]), am, bl)) * (1.0 + 1e-15);
            const double db = fma(-G2 * G2, rd2[p], c1);
            const double wb = fma(G2, as2[p], w1) * (1.0 + 1e-14);
            const double q = fma(wb, wb, bm[p]);
            need |= !(db > 1e-6 && fma(kq[p], db, -q) > 0.0);
        }
        if (__any_sync(L0S_FULL, need)) word |= 1u << bb;
    }
    return word;
}

#ifndef L0S_TSK4
#define L0S_TSK4 1
#endif
constexpr bool TSK4 = L0S_TSK4;
// SCR: the screened instantiation (launched first; each CTA runs the one its threshold selects,
// as in fit3.cu's k_fit3).
template <int NT, bool SCR>
__global__ void __launch_bounds__(256, 1) k_fit4(const __grid_constant__ FitArgs a) {
    using C = Cfg4<NT>;
    constexpr int P = C::P, IB = C::IB, TS = C::TS, BS = C::BS, LSPAN = C::LSPAN;
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_unit;
    __shared__ unsigned char s_force[2][IB];
    __shared__ unsigned s_need;
    __shared__ int s_use;
    int t0 = -1;                      // SCR: the screened task slot
    unsigned long long n_tests = 0;   // SCR: tile tests of this warp (flushed at the end)
    if constexpr (TSK4) {
        if (threadIdx.x == 0) {
            double y2 = 0.0;
            for (int t = 0; t < a.T; ++t) y2 = fmax(y2, a.G[(int64_t)t * a.mp * a.mp + a.m * a.mp + a.m]);
            const double th = a.collect == 1 ? a.theta0 : ord_dec(*(volatile unsigned long long*)a.theta_g);
            int tt = -1;
            if (a.tmax) {
                const int64_t nbk = (a.m + IB - 1) / IB;
                tt = (int)a.tmax[(a.m + 1 + (a.m + 31) / 32) * nbk];
            }
            s_use = (a.tmax != nullptr && th < y2 && tt >= 0 && tt < NT) ? tt : -1;
        }
        __syncthreads();
        if ((s_use >= 0) != SCR) return;
        t0 = s_use;
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double* sKraw = sm + 2 * BS + 2 * NW * CAP_WIDE + tid * P;
    const int64_t m = a.m, mp = a.mp;
    const double shrink = (NT == 1) ? 1.0 : (1.0 - 2.0 * kRcpRel);
    WarpCands wc{sm + 2 * BS + warp * CAP_WIDE, reinterpret_cast<int64_t*>(sm + 2 * BS + NW * CAP_WIDE) + warp * CAP_WIDE, 0,
                 a.collect == 1 ? a.theta0 : ord_dec(*(volatile unsigned long long*)a.theta_g), 0, CAP_WIDE};
    const int64_t* B2 = a.binom + 2 * (m + 1);
    const int64_t* B3 = a.binom + 3 * (m + 1);
    const int64_t* B4 = a.binom + 4 * (m + 1);

    auto load_tiles = [&](int buf, int ib0, int j0, int k, int l0) {
        double* base = sm + buf * BS;
        if (tid < IB) s_force[buf][tid] = (ib0 + tid < m) ? a.iforce[ib0 + tid] : 0;
        constexpr int pr = 16 + LSPAN / 2 + 2;  // 16-byte pieces for j and l, then C[i,k] and c_i
        for (int q = tid; q < NT * IB * pr; q += 256) {
            const int t = q / (IB * pr), r = q % (IB * pr);
            const int row = r / pr, piece = r % pr;
            const double* Grow = a.G + (int64_t)t * mp * mp + (int64_t)(ib0 + row) * mp;
            double* Tt = base + t * TS;
            if (piece < 16)
                cp_async16(Tt + row * 32 + piece * 2, Grow + j0 + piece * 2);
            else if (piece < 16 + LSPAN / 2)
                cp_async16(Tt + IB * 32 + row * LSPAN + (piece - 16) * 2, Grow + l0 + (piece - 16) * 2);
            else if (piece == 16 + LSPAN / 2)
                cp_async8(Tt + IB * (32 + LSPAN) + row, Grow + k);
            else
                cp_async8(Tt + IB * (33 + LSPAN) + row, Grow + m);
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
        const int j0 = (U.x & 0xffff) * 32, l0 = (U.x >> 16) * LSPAN;
        const int k = U.y;
        const int j = j0 + lane;
        const int lbase = l0 + warp * P;
        const int i_lo = U.z, i_hi = U.w;
        load_tiles(0, i_lo, j0, k, l0);
        if (a.collect != 1) {
            // shared threshold: the global bound histogram and the other warps' lists
            double th = fmin(hist_theta(a, lane), ord_dec(*(volatile unsigned long long*)a.theta_g));
            if (th < wc.theta) {
                wc.theta = th;
                if (lane == 0) atomicMin(a.theta_g, ord_enc(th));
            }
        }

        // ---------------- hoist ----------------
        double L10[NT], rd1[NT], s1[NT], w0[NT];
        double L20[P][NT], L21[P][NT], rd2[P][NT], s2[P][NT], Kq[P], Bm[P];
        double K0[SCR ? P : 1];  // SCR: slot t0's share of the bound, base_t0 - A_t0
        unsigned valid = 0, bad = 0, forced = 0;
        const int jj = j < m ? j : (int)m - 1;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int l = lbase + p;
            const int ll = l < m ? l : (int)m - 1;
            double kr = 0.0, bm = 0.0;
            bool isbad = false, isnan_ = false;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double* Gt = a.G + (int64_t)t * mp * mp;
                const double Y2 = Gt[m * mp + m];
                const Hoist3 h = hoist3(Gt, mp, m, j, k, l);
                double At, Bt, vk;
                const double* rt_ = a.rho + (int64_t)t * m;
                const double rh = fmax(fmax(a.rho_cap[t], rt_[jj]), fmax(rt_[k], rt_[ll]));
                task_bound(4, a.eta[t], ref_gamma(a.rowsd[t], 4, a.ref_fp32), rh, Y2, a.ynorm[t], h.tr3, At, Bt, vk);
                L10[t] = h.L10;
                rd1[t] = h.rd1;
                s1[t] = h.s1;
                w0[t] = h.w0;
                L20[p][t] = h.L20;
                L21[p][t] = h.L21;
                rd2[p][t] = h.rd2;
                s2[p][t] = h.s2;
                kr += h.base - At;
                if constexpr (SCR) {
                    if (t == t0) K0[p] = h.base - At;
                }
                bm = fmax(bm, Bt);
                if (!(h.d1 > 0.0) || !(h.d2 > 0.0) || !(vk * (1.0 + 4.0 * h.tr3) <= FO_LIM)) isbad = true;
                // dead features (NaN Gram rows) drop the pair; a NaN produced by a near-singular
                // (j, k, l) block (d1 or d2 <= 0) is `bad` and goes to the exact kernel instead
                const double raw = h.w0 + h.L10 + h.L20 + Gt[l * mp + k] + Gt[m * mp + k] + Gt[m * mp + l];
                if (raw != raw) isnan_ = true;
            }
            sKraw[p] = kr;
            Bm[p] = bm;
            if (j < k && k < l && l < m && !isnan_) valid |= 1u << p;
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

        // ---------------- tile screen (SCR) ----------------
        const int nib = (i_hi - i_lo + IB - 1) / IB;
        unsigned wneed = ~0u, cneed = ~0u;  // this warp's / the CTA's needed tiles
        if constexpr (SCR) {
            if (tid == 0) s_need = 0u;
            __syncthreads();
            if (nib <= 32) {
                Slot4 h4;
                double l20[P], l21[P], r2[P], a2[P], kq[P];
                unsigned cand = 0u;
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    if (t == t0) {
                        h4.la10 = fabs(L10[t]);
                        h4.rd1 = rd1[t] * (1.0 + 2e-14);
                        h4.as1 = fabs(s1[t]);
                        h4.aw0 = fabs(w0[t]);
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            l20[p] = L20[p][t];
                            l21[p] = L21[p][t];
                            r2[p] = rd2[p][t] * (1.0 + 2e-14);
                            a2[p] = fabs(s2[p][t]);
                        }
                    }
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double x = (NT == 1) ? Kq[p] : (K0[p] - wc.theta) * shrink;
                    kq[p] = x * (1.0 / ((1.0 + 4.0 * kRcpRel) * (1.0 + 1e-12)));
                    if (!((forced >> p) & 1u) && kq[p] > 0.0) cand |= 1u << p;
                }
                wneed = tile_screen4<P, IB>(a, h4, l20, l21, r2, a2, kq, Bm, valid, cand, lane, U.x & 0xffff, k,
                                            lbase, i_lo, i_hi, nib);
                n_tests += (unsigned long long)nib;
            }
            if (lane == 0) atomicOr(&s_need, wneed);
            __syncthreads();
            cneed = __reduce_or_sync(L0S_FULL, s_need);  // (warp-uniform for the compiler)
        }
        // needed tiles in order; tile 0 was staged before the hoist
        auto next_tile = [&](int b) -> int {
            if constexpr (SCR) {
                const unsigned mk = b >= 32 ? 0u : (cneed & (~0u << b));
                return (b < 32 && mk) ? (__ffs(mk) - 1) : nib;
            } else {
                return b;
            }
        };
        int bi = next_tile(0);
        if (SCR && bi != 0) {
            cp_async_wait<0>();  // tile 0's copies land before buffer 0 is refilled
            __syncthreads();
            if (bi < nib) load_tiles(0, i_lo + bi * IB, j0, k, l0);
        }

        // ---------------- sweep i ----------------
        for (int buf = 0; bi < nib; buf ^= 1) {
            const int ib0 = i_lo + bi * IB;
            const int bn = next_tile(bi + 1);
            if (bn < nib) {
                load_tiles(buf ^ 1, i_lo + bn * IB, j0, k, l0);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const double* T0 = sm + buf * BS;
            constexpr int NPW = (IB * P + 31) / 32;
            constexpr int IPW = 32 / P;
            unsigned pend[NPW];
            const bool wn = !SCR || __any_sync(L0S_FULL, (wneed >> (bi & 31)) & 1u);
#pragma unroll
            for (int pw = 0; pw < NPW; ++pw) {
                unsigned word = 0u;
#pragma unroll 1
                for (int iw = 0; iw < (wn ? IPW : 0); ++iw) {
                    const int ii = pw * IPW + iw;
                    const int i = ib0 + ii;
                    double acc[P];
#pragma unroll
                    for (int p = 0; p < P; ++p) acc[p] = Kq[p];
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        const double* Tt = T0 + t * TS;
                        const double g0 = Tt[ii * 32 + lane];
                        const double gkk = Tt[IB * (32 + LSPAN) + ii];
                        const double ci = Tt[IB * (33 + LSPAN) + ii];
                        const double D = fma(-g0, g0, 1.0);
                        const double V = fma(-g0, w0[t], ci);
                        const double g1 = fma(-L10[t], g0, gkk);
                        const double t1 = g1 * rd1[t];
                        const double D1 = fma(-t1, g1, D);
                        const double V1 = fma(-g1, s1[t], V);
                        double gl[P];
#pragma unroll
                        for (int p = 0; p < P; p += 2) {
                            const double2 v =
                                *reinterpret_cast<const double2*>(Tt + IB * 32 + ii * LSPAN + warp * P + p);
                            gl[p] = v.x;
                            gl[p + 1] = v.y;
                        }
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            const double g2 = fma(-L21[p][t], g1, fma(-L20[p][t], g0, gl[p]));
                            const double t2 = g2 * rd2[p][t];
                            const double w = fma(-g2, s2[p][t], V1);
                            const double d = fma(-t2, g2, D1);
                            const double q = fma(w, w, Bm[p]);
                            if (NT == 1)
                                acc[p] = fma(acc[p], d, -q);
                            else
                                acc[p] = fma(-q, fabs(rcp_sweep(d)), acc[p]);
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
                    const int i = ib0 + ii, l = lbase + p;
                    *rkv = a.N_total - 1 - (B4[m - 1 - i] + B3[m - 1 - j] + B2[m - 1 - k] + (m - 1 - l));
                    if (a.ranged && (*rkv < a.rank_lo || *rkv >= a.rank_hi)) return 0;
                    if ((bad >> p) & 1u) return 2;
                    return eval_tuple4(a, i, j, k, l, lbv) == 3 ? 1 : 2;
                },
                set_kq);
            __syncthreads();
            bi = bn;
        }
    }
    if (SCR && lane == 0 && n_tests && a.n_screen) atomicAdd(a.n_screen, n_tests);
    flush_warp(a, wc, blockIdx.x * NW + warp, lane);
}

__global__ void k_screen4(const __grid_constant__ FitArgs a, const int64_t* __restrict__ tuples, int64_t count,
                          double* __restrict__ out_lb, int32_t* __restrict__ out_flags) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    double lb;
    out_flags[c] = eval_tuple4(a, tuples[4 * c], tuples[4 * c + 1], tuples[4 * c + 2], tuples[4 * c + 3], &lb);
    out_lb[c] = lb;
}

template <int NT>
int occupancy4(int nsm) {
    using C = Cfg4<NT>;
    cudaFuncSetAttribute(k_fit4<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes);
    cudaFuncSetAttribute(k_fit4<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit4<NT, false>, 256, C::smem_bytes);
    return nsm * (per_sm < 1 ? 1 : per_sm);
}

__global__ void __launch_bounds__(128) k_seed_eval4(const __grid_constant__ FitArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= *a.seed_n) return;
    double lb = 0.0, ub = INFINITY;
    const int fl = a.seed_tup[c * kSeedW] >= 0 ? eval_tuple4(a, a.seed_tup[c * kSeedW + 0], a.seed_tup[c * kSeedW + 1], a.seed_tup[c * kSeedW + 2], a.seed_tup[c * kSeedW + 3], &lb, &ub) : 0;
    a.seed_ub[c] = (fl == 3 && ub == ub) ? ub : INFINITY;
}

template <int NT>
int launch4(const FitArgs& a, int nsm, cudaStream_t st) {
    const int grid = occupancy4<NT>(nsm);
    if (a.collect != 1) seed_launch<4, 12>(k_seed_eval4, a, st);
    if (TSK4 && a.tmax) {
        k_tile_max<Cfg4<NT>::IB><<<dim3((unsigned)((a.m + 256) / 256), (unsigned)((a.m + Cfg4<NT>::IB - 1) / Cfg4<NT>::IB)),
                                    256, 0, st>>>(a.G, a.iforce, a.m, a.mp, a.T, a.tmax);
        k_fit4<NT, true><<<grid, 256, Cfg4<NT>::smem_bytes, st>>>(a);
    }
    k_fit4<NT, false><<<grid, 256, Cfg4<NT>::smem_bytes, st>>>(a);
    return grid;
}

}  // namespace

void launch_screen4(const FitArgs& a, const int64_t* tuples, int64_t count, double* out_lb, int32_t* out_flags,
                    cudaStream_t st) {
    if (count > 0) k_screen4<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(a, tuples, count, out_lb, out_flags);
}

int fit4_lspan(int T) { return T <= 2 ? Cfg4<1>::LSPAN : Cfg4<8>::LSPAN; }

int fit4_grid(int T, int nsm) {
    switch (T) {
        case 1: return occupancy4<1>(nsm);
        case 2: return occupancy4<2>(nsm);
        case 3: return occupancy4<3>(nsm);
        case 4: return occupancy4<4>(nsm);
        case 5: return occupancy4<5>(nsm);
        case 6: return occupancy4<6>(nsm);
        case 7: return occupancy4<7>(nsm);
        case 8: return occupancy4<8>(nsm);
        default: return T > 8 ? occupancy4<8>(nsm) : -1;
    }
}

int fit4_launch(const FitArgs& a, int nsm, cudaStream_t st) {
    switch (a.T) {
        case 1: return launch4<1>(a, nsm, st);
        case 2: return launch4<2>(a, nsm, st);
        case 3: return launch4<3>(a, nsm, st);
        case 4: return launch4<4>(a, nsm, st);
        case 5: return launch4<5>(a, nsm, st);
        case 6: return launch4<6>(a, nsm, st);
        case 7: return launch4<7>(a, nsm, st);
        case 8: return launch4<8>(a, nsm, st);
        default: return a.T > 8 ? launch4<8>(a, nsm, st) : -1;  // T > 8: the first 8 tasks bound the sweep
    }
}

// Unit table for n = 4: (j-block | l-block << 16, k, i_lo, i_hi) with i < j < k < l < m.
// c3_prefix[v] = rank of the first tuple whose smallest index is v.
std::vector<int4> fit4_units(int64_t m, int T, const std::vector<int64_t>& c3_prefix, int64_t rank_lo,
                             int64_t rank_hi) {
    const int lspan = fit4_lspan(T);
#ifndef L0S_ICH4
#define L0S_ICH4 512  // i rows per unit (C4: 128 -> 512, plain sweep 86 -> 77 ms, screened 42 -> 22 ms)
#endif
    const int ich = L0S_ICH4;
    std::vector<int4> units;
    const int nJ = (int)((m + 31) / 32);
    const int nL = (int)((m + lspan - 1) / lspan);
    int i_first = 0, i_last = (int)m - 1;
    while (i_first < m && c3_prefix[i_first + 1] <= rank_lo) ++i_first;
    while (i_last > 0 && c3_prefix[i_last] >= rank_hi) --i_last;
    for (int jb = 0; jb < nJ; ++jb) {
        const int jlo = jb * 32;
        int i_end = (int)std::min<int64_t>(jlo + 31, m - 3);
        i_end = std::min(i_end, i_last + 1);
        if (i_end <= i_first) continue;
        for (int k = jlo + 1; k <= m - 2; ++k) {
            for (int lb = (k + 1) / lspan; lb < nL; ++lb) {
                if ((int64_t)lb * lspan + lspan - 1 <= k) continue;
                for (int lo = i_first; lo < i_end; lo += ich) {
                    const int hi = std::min(lo + ich, i_end);
                    if (c3_prefix[hi] <= rank_lo || c3_prefix[lo] >= rank_hi) continue;
                    units.push_back(make_int4(jb | (lb << 16), k, lo, hi));
                }
            }
        }
    }
    std::stable_sort(units.begin(), units.end(),
                     [](const int4& x, const int4& y) { return (x.w - x.z) > (y.w - y.z); });
    return units;
}

}  // namespace l0s
