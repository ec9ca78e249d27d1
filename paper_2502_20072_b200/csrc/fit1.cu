// fit1.cu -- screened fit of every 1-tuple (one feature), fp64 / fp32 reference rounding.
//
// The dimension-1 member of the screened family (fit2/3/4.cu), for the reference's
// score_tuples (lsq.py:113-156) at n = 1: with the centered, unit-norm feature z_f and
// c_f = z_f . y_c (the staged Gram's property row), the task SSR is |y_c|^2 - c_f^2.
// There are only m tuples, so no sweep or threshold machinery is needed: one thread per
// feature writes the rigorous lower bound of fitcommon.cuh (n = 1: the hoisted block is
// empty, trace 0, the new pivot d = 1, so tr(C^-1) = 1) to a dense list, which the host
// sorts and refits in order until the keep-th exact score is certified (api.cu,
// search_fast1).  A feature whose bound is not trustworthy, or whose rank-rule certificate
// fails, goes to the ill list (QR screen + bit-exact refit); a dead feature (NaN Gram row:
// the reference rejects every tuple holding it) gets +inf.
#include "fitcommon.cuh"

namespace l0s {

using namespace fit;

namespace {

__global__ void __launch_bounds__(256) k_fit1(const __grid_constant__ FitArgs a, int64_t rb, int64_t re,
                                              double* __restrict__ out_lb, int64_t* __restrict__ out_rank) {
    const int64_t f = rb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= re) return;
    const int64_t m = a.m, mp = a.mp;
    double lb = 0.0;
    bool cond = true, rank_ok = true, dead = false;
    for (int t = 0; t < a.T; ++t) {
        const double* Gt = a.G + (int64_t)t * mp * mp;
        const double Y2 = Gt[m * mp + m];
        const double c = Gt[m * mp + f];
        double At, Bt, vk;
        task_bound(1, a.eta[t], ref_gamma(a.rowsd[t], 1, a.ref_fp32), a.rho[(int64_t)t * m + f], Y2, a.ynorm[t], 0.0,
                   At, Bt, vk);
        if (!(vk * 2.0 <= FO_LIM) || !(At + Bt <= (a.ref_fp32 ? LOOSE32 : LOOSE) * Y2)) cond = false;
        if (c != c) dead = true;
        lb += fma(-c, c, Y2) - At - Bt;
        const int64_t f1[1] = {f};
        if (!rank_certain<1>(a, t, f1, 1.0)) rank_ok = false;
    }
    const int64_t i = f - rb;
    out_rank[i] = f;  // the rank of the 1-tuple (f) is f (search.py:66-104)
    if (dead) {
        out_lb[i] = INFINITY;
    } else if (cond && rank_ok) {
        out_lb[i] = lb;
    } else {
        out_lb[i] = INFINITY;  // sorted last; scored through the ill list instead
        const unsigned long long x = atomicAdd(a.ill_cnt, 1ull);
        if ((int64_t)x < a.ill_cap) a.ill[x] = f;
    }
}

}  // namespace

void launch_fit1(const FitArgs& a, int64_t rb, int64_t re, double* out_lb, int64_t* out_rank, cudaStream_t st) {
    if (re > rb) k_fit1<<<(unsigned)((re - rb + 255) / 256), 256, 0, st>>>(a, rb, re, out_lb, out_rank);
}

}  // namespace l0s
