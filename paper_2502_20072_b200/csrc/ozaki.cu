// ozaki.cu -- the per-task Gram on the INT8 tensor cores (tcgen05.mma kind::i8, TMEM).
//
// Ozaki splitting: every row f of Z (one task's segment) is scaled by 2^-e_f (max |z| < 2^e_f)
// and cut into S = 4 signed 7-bit digits, u = sum_a q_a 2^-7a + rho, |q_a| <= 127,
// |rho| < 2^-28.  Then
//     G[f, g] = 2^(e_f + e_g) sum_{a + b <= S + 1} 2^-7(a+b) sum_s q_fa(s) q_gb(s)  (+ error)
// where every inner sum is an exact int32 (|.| <= 4 r 127^2 < 2^31 for r <= 33k samples):
// the tensor cores accumulate it in TMEM, one accumulator per digit weight d = a + b
// (4 x 128 columns), and the epilogue combines the four in fp64.  The dropped digit
// products and the remainders bound the error of every entry by
//     eta_t = C4 r_t max_f 2^(2 e_f)   (C4 = 1.9e-8, normalised to unit rows)
// which the screen's error model takes in place of the fp64 dot-product bound; a task whose
// eta exceeds OZ_ETA_MAX falls back to the DMMA Gram (spiky rows).
//
// GEMM: one CTA per 128 x 128 upper-triangle tile of one task, one CTA per SM (all 512 TMEM
// columns: four 128-column accumulators, one per digit weight; 64-wide tiles with two CTAs per
// SM were 6 % slower); 192 threads = TMA producer warp, MMA warp (one elected thread issues
// tcgen05.mma; it also owns the TMEM allocation) and 4 epilogue warps (tcgen05.ld by TMEM lane
// quadrant, stores staged through shared memory so both G[r][c] and its mirror G[c][r] are
// coalesced).  A pipeline stage is one 64-byte K chunk of all 4 digit planes of both operands
// (8 TMA boxes, SWIZZLE_64B, 64 KB), 3 stages; each stage feeds 10 digit pairs x 2 MMAs of
// 128 x 128 x 32.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {

constexpr int OZ_S = OZ_DIGITS;     // digits per value (kernels.h: the normalize kernel writes them)
constexpr int OZ_NG = OZ_S;         // digit-weight groups d = 2 .. S + 1
constexpr int OZ_BM = 128;          // tile rows (TMEM lanes)
#ifndef L0S_OZ_BN
#define L0S_OZ_BN 128
#endif
// tile cols: 4 groups x 128 = all 512 TMEM columns (one CTA per SM, N = 128 MMAs run at the
// full rate); 64 gives two CTAs per SM with half-width MMAs
constexpr int OZ_BN = L0S_OZ_BN;
constexpr int OZ_KC = 64;           // K bytes per stage
constexpr int OZ_ST = OZ_BN >= 128 ? 3 : 2;  // stages per CTA
constexpr int OZ_CTAS = OZ_BN >= 128 ? 1 : 2;  // CTAs per SM (TMEM)
constexpr int OZ_TA = OZ_BM * OZ_KC;                // 8 KB: one digit plane of A
constexpr int OZ_TB = OZ_BN * OZ_KC;                // 4 KB: one digit plane of B
constexpr int OZ_STAGE = OZ_S * (OZ_TA + OZ_TB);    // 48 KB
constexpr int OZ_SMEM = OZ_ST * OZ_STAGE + 1024;    // + alignment slack
constexpr int OZ_TMEM_COLS = OZ_NG * OZ_BN;         // 512 (256 for 64-wide tiles)
constexpr double OZ_C = 1.9e-8;     // error constant per unit-scaled entry and sample (S = 4)

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major operand tile, rows of 64 bytes, 64-byte swizzle: 8-row atoms of 512 B
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);  // start address
    d |= (uint64_t)1 << 16;                    // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;           // stride byte offset: 8 rows x 64 B
    d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;                    // SWIZZLE_64B
    return d;
}

// kind::i8 instruction descriptor: s32 accumulate, s8 x s8, K-major A and B, M = 128, N = 64
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(OZ_IDESC), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
            "r"(smem_addr(dst)),
        "l"(reinterpret_cast<unsigned long long>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
        : "memory");
}

// ---- digits: one warp per (row f < mp, task t) ----
__global__ void k_oz_split(const double* __restrict__ Z, int64_t sp, const int64_t* __restrict__ zoff, int T, int64_t mp,
                           int64_t R, const int64_t* __restrict__ koff, int8_t* __restrict__ Q, int64_t KP,
                           int* __restrict__ ex) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= mp * T) return;
    const int t = (int)(wid % T);
    const int64_t f = wid / T;
    const double* src = Z + f * sp + zoff[t];
    const int len = (int)(zoff[t + 1] - zoff[t]);
    const int64_t k0 = koff[t];
    const int klen = (int)(koff[t + 1] - k0);
    double mx = 0.0;
    for (int j = lane; j < len; j += 32) mx = fmax(mx, fabs(src[j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(L0S_FULL, mx, o));
    // e: max |z| < 2^e (exact power-of-two scaling); NaN rows (dead features) give zero digits
    int e = 0;
    if (mx > 0.0 && mx == mx && mx < INFINITY) {
        frexp(mx, &e);  // mx = m 2^e, 0.5 <= m < 1
    }
    for (int j = lane; j < klen; j += 32) {
        double u = (j < len && mx == mx) ? ldexp(src[j], -e) : 0.0;
        if (!(u == u)) u = 0.0;
#pragma unroll
        for (int a = 0; a < OZ_S; ++a) {
            const double v = u * 128.0;  // exact
            const double q = trunc(v);   // |q| <= 127
            u = v - q;                   // exact remainder
            Q[((int64_t)a * R + f) * KP + k0 + j] = (int8_t)(int)q;
        }
    }
    if (lane == 0) ex[(int64_t)t * R + f] = e;
}

// ---- GEMM: one OZ_BM x OZ_BN tile (rows fb, cols gb, fb * OZ_BM <= the block's last column:
// every entry with row <= col lies in exactly one such tile) of one task per CTA ----
// Tiles are numbered column by column (gb outer, fb = 0 .. inner) from tile g0, so a range of
// column blocks -- the part of the Gram a landed row chunk completes -- is one launch.
// tiles of column block gb: row blocks fb with fb * BM <= the block's last column
__host__ __device__ constexpr int oz_tiles_in_block(int gb) { return ((gb + 1) * OZ_BN - 1) / OZ_BM + 1; }

__global__ void __launch_bounds__(192, OZ_CTAS) k_oz_gemm(const __grid_constant__ TmaDesc tmA,
                                                   const __grid_constant__ TmaDesc tmB, const int64_t* __restrict__ koff,
                                                   const int* __restrict__ ex, int64_t R, int nbc, int64_t mp,
                                                   double* __restrict__ Gall, int g0) {
    extern __shared__ unsigned char oz_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)oz_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) unsigned long long full[OZ_ST], empty[OZ_ST], done;
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.y;
    int lin = g0 + blockIdx.x, gb = 0;
    while (lin >= oz_tiles_in_block(gb)) {
        lin -= oz_tiles_in_block(gb);
        ++gb;
    }
    const int fb = lin;
    const int64_t k0 = koff[t];
    const int nkc = (int)((koff[t + 1] - k0) / OZ_KC);
    if (threadIdx.x == 0) {
        for (int s = 0; s < OZ_ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&tmem_slot)),
                     "r"(OZ_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            for (int kc = 0; kc < nkc; ++kc) {
                const int s = kc % OZ_ST;
                if (kc >= OZ_ST) mbar_wait(&empty[s], (unsigned)((kc / OZ_ST - 1) & 1));
                unsigned char* st = sm + s * OZ_STAGE;
                mbar_expect_tx(&full[s], (unsigned)OZ_STAGE);
                const int x = (int)(k0 + (int64_t)kc * OZ_KC);
                for (int a = 0; a < OZ_S; ++a) {
                    tma_load_3d(st + a * OZ_TA, &tmA, x, fb * OZ_BM, a, &full[s]);
                    tma_load_3d(st + OZ_S * OZ_TA + a * OZ_TB, &tmB, x, gb * OZ_BN, a, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            for (int kc = 0; kc < nkc; ++kc) {
                const int s = kc % OZ_ST;
                mbar_wait(&full[s], (unsigned)((kc / OZ_ST) & 1));
                tc_fence_after();
                const uint32_t st = smem_addr(sm + s * OZ_STAGE);
#pragma unroll
                for (int a = 1; a <= OZ_S; ++a)
#pragma unroll
                    for (int b = 1; a + b <= OZ_S + 1; ++b)
#pragma unroll
                        for (int kk = 0; kk < OZ_KC / 32; ++kk) {
                            const uint64_t da = sw64_desc(st + (a - 1) * OZ_TA + kk * 32);
                            const uint64_t db = sw64_desc(st + OZ_S * OZ_TA + (b - 1) * OZ_TB + kk * 32);
                            const uint32_t acc = (kc == 0 && kk == 0 && a == 1) ? 0u : 1u;
                            mma_i8(tmem + (uint32_t)(a + b - 2) * OZ_BN, da, db, acc);
                        }
                mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
            }
            mma_commit(&done);
        }
    } else {  // epilogue warps 2..5: TMEM lane quadrant (warp % 4) = 32 tile rows
        mbar_wait(&done, 0u);
        tc_fence_after();
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const int64_t row0 = (int64_t)fb * OZ_BM + quad * 32;
        const int64_t row = row0 + lane;
        const int er = ex[(int64_t)t * R + row];
        double* G = Gall + (int64_t)t * mp * mp;
        // staging for coalesced row stores: this warp's 32 rows x 32 cols (stage buffers are idle now)
        double* stg = reinterpret_cast<double*>(sm) + quad * 32 * 33;
        // the tile's column scales 2^e_c, once per warp in shared memory behind the staging area
        // (e_f + e_g >= -1022 for unit rows: 2^e_f 2^e_g is exact, and acc * 2^(e_f + e_g) is the
        // same single rounding ldexp performs)
        double* csc = reinterpret_cast<double*>(sm) + 4 * 32 * 33 + quad * OZ_BN;
        for (int c = lane; c < OZ_BN; c += 32) csc[c] = ldexp(1.0, ex[(int64_t)t * R + (int64_t)gb * OZ_BN + c]);
        const double rsc = ldexp(1.0, er);
        __syncwarp();
        for (int c0 = 0; c0 < OZ_BN; c0 += 32) {
            double acc[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll
            for (int g = 0; g < OZ_NG; g += 2) {  // two accumulators per wait
                uint32_t v[2][32];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)((g + h) * OZ_BN + c0);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                        : "=r"(v[h][0]), "=r"(v[h][1]), "=r"(v[h][2]), "=r"(v[h][3]), "=r"(v[h][4]), "=r"(v[h][5]),
                          "=r"(v[h][6]), "=r"(v[h][7]), "=r"(v[h][8]), "=r"(v[h][9]), "=r"(v[h][10]), "=r"(v[h][11]),
                          "=r"(v[h][12]), "=r"(v[h][13]), "=r"(v[h][14]), "=r"(v[h][15]), "=r"(v[h][16]),
                          "=r"(v[h][17]), "=r"(v[h][18]), "=r"(v[h][19]), "=r"(v[h][20]), "=r"(v[h][21]),
                          "=r"(v[h][22]), "=r"(v[h][23]), "=r"(v[h][24]), "=r"(v[h][25]), "=r"(v[h][26]),
                          "=r"(v[h][27]), "=r"(v[h][28]), "=r"(v[h][29]), "=r"(v[h][30]), "=r"(v[h][31])
                        : "r"(taddr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double w = ldexp(1.0, -7 * (g + h + 2));
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc[j] = fma((double)(int)v[h][j], w, acc[j]);  // exact products
                }
            }
            const int64_t col0 = (int64_t)gb * OZ_BN + c0;
#pragma unroll
            for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = acc[j] * (rsc * csc[c0 + j]);
            __syncwarp();
            // rows of the warp, lanes over columns: G[row][col] for row <= col, coalesced
            const int64_t col = col0 + lane;
            for (int i = 0; i < 32; ++i) {
                const int64_t rw = row0 + i;
                if (rw < mp && col < mp && rw <= col) G[rw * mp + col] = stg[i * 33 + lane];
            }
            // mirror: columns of the chunk, lanes over rows: G[col][row], coalesced
            for (int j = 0; j < 32; ++j) {
                const int64_t cl = col0 + j;
                if (row < mp && cl < mp && row <= cl) G[cl * mp + row] = stg[lane * 33 + j];
            }
            __syncwarp();
        }
        (void)r;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZ_TMEM_COLS));
    }
}

// eta_t = C r_t max over rows of 2^(2 e) / |row|^2 (features: unit rows; the property row: Y2)
// eta_t = C r_t max_f 2^(2 e_f) (the property row relative to |y_c|^2).  With a fix-up list
// (rows != nullptr), rows whose own term exceeds `lim` in some task are loose: listed (any order:
// k_oz_fixup's result does not depend on it), counted, and left out of the maximum, which is
// floored at the fp64 dot-product bound their recomputed entries carry.  One CTA.
__global__ void __launch_bounds__(1024) k_oz_eta(const int* __restrict__ ex, int64_t R, int T, int64_t m, int64_t mp,
                                                 const double* __restrict__ Gall, const double* __restrict__ rows,
                                                 double lim, double* __restrict__ eta, int* __restrict__ fix_rows,
                                                 int* __restrict__ fix_count, int fix_cap,
                                                 unsigned char* __restrict__ s_loose) {  // (m + 1,) when fixing up
    __shared__ double red[32];
    __shared__ int s_cnt;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    auto term = [&](int t, int64_t f) {
        double v = ldexp(1.0, 2 * ex[(int64_t)t * R + f]);
        if (f == m) {
            const double y2 = Gall[(int64_t)t * mp * mp + m * mp + m];
            v = y2 > 0.0 ? v / y2 : 0.0;
        }
        return OZ_C * rows[t] * v * (1.0 + 1e-6);
    };
    const bool fixing = fix_rows != nullptr;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    if (fixing) {
        for (int64_t f = tid; f <= m; f += blockDim.x) {
            bool loose = false;
            for (int t = 0; t < T && !loose; ++t) loose = !(term(t, f) <= lim);
            s_loose[f] = loose;  // global: read back below by this CTA only (after the barrier)
            if (loose) {
                const int k = atomicAdd(&s_cnt, 1);
                if (k < fix_cap) fix_rows[k] = (int)f;
            }
        }
        __syncthreads();
    }
    for (int t = 0; t < T; ++t) {
        double mx = 0.0;
        for (int64_t f = tid; f <= m; f += blockDim.x)
            if (!fixing || !s_loose[f]) mx = fmax(mx, term(t, f));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(L0S_FULL, mx, o));
        if (lane == 0) red[warp] = mx;
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nw; ++w) mx = fmax(mx, red[w]);
            eta[t] = fixing ? fmax(mx, 4.0 * (rows[t] + 8.0) * 1.1102230246251565e-16) : mx;
        }
        __syncthreads();
    }
    if (tid == 0 && fix_count) *fix_count = fixing ? s_cnt : 0;
}

// fp64 Gram entries G[t][f][g] = G[t][g][f] = sum_i z_f(i) z_g(i) of the loose rows f (k_oz_eta's
// list) against every row g <= m, z = (x - mean) * scale exactly as the staging kernel computed
// the digits' values (mean, scale stored beside them).  CTA: one task, FX loose rows staged in
// shared memory chunk by chunk, FG rows g per warp (lanes stride the samples, FG x FX fp64
// accumulators per lane, warp sums at the end).
constexpr int FX = 8, FG = 4, FCH = 256, FTH = 256;
template <typename W>
__global__ void __launch_bounds__(FTH) k_oz_fixup(const W* __restrict__ Xp, const W* __restrict__ yp, int64_t m, int64_t s,
                                                  const int64_t* __restrict__ bounds, const double* __restrict__ musc,
                                                  int64_t R, int64_t mp, const int* __restrict__ fix_rows,
                                                  const int* __restrict__ fix_count, int fix_cap, double* __restrict__ G) {
    const int nl = *fix_count;
    if (nl == 0 || nl > fix_cap) return;  // none, or too many: the host then recomputes the Gram on DMMA
    __shared__ double zf[FX][FCH];
    __shared__ double fms[FX][2];
    __shared__ int frow[FX];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.y;
    const int64_t lo = bounds[t], r = bounds[t + 1] - lo;
    const double* ms = musc + 2 * (int64_t)t * R;
    for (int l0 = 0; l0 < nl; l0 += FX) {  // batches of FX loose rows
        __syncthreads();  // the previous batch's frow / fms / zf reads are done
        if (tid < FX) {
            const int f = l0 + tid < nl ? fix_rows[l0 + tid] : -1;
            frow[tid] = f;
            fms[tid][0] = f >= 0 ? ms[2 * f] : 0.0;
            fms[tid][1] = f >= 0 ? ms[2 * f + 1] : 0.0;
        }
        const int64_t g0 = ((int64_t)blockIdx.x * (FTH / 32) + warp) * FG;
        double gmu[FG], gsc[FG];
        const W* grow[FG];
    #pragma unroll
        for (int q = 0; q < FG; ++q) {
            const int64_t g = g0 + q <= m ? g0 + q : m;
            gmu[q] = ms[2 * g];
            gsc[q] = ms[2 * g + 1];
            grow[q] = (g < m ? Xp + g * s : yp) + lo;
        }
        double acc[FG][FX];
    #pragma unroll
        for (int q = 0; q < FG; ++q)
    #pragma unroll
            for (int l = 0; l < FX; ++l) acc[q][l] = 0.0;
        for (int64_t c0 = 0; c0 < r; c0 += FCH) {
            __syncthreads();  // frow / fms (first chunk), the previous chunk's reads (later ones)
            for (int x = tid; x < FX * FCH; x += FTH) {
                const int l = x / FCH, i = x % FCH;
                const int f = frow[l];
                double z = 0.0;
                if (f >= 0 && c0 + i < r) {
                    const W* src = (f < m ? Xp + (int64_t)f * s : yp) + lo;
                    z = ((double)src[c0 + i] - fms[l][0]) * fms[l][1];
                }
                zf[l][i] = z;
            }
            __syncthreads();
    #pragma unroll
            for (int k = 0; k < FCH / 32; ++k) {
                const int i = k * 32 + lane;
                const bool in = c0 + i < r;
                double zf_[FX];
    #pragma unroll
                for (int l = 0; l < FX; ++l) zf_[l] = zf[l][i];
    #pragma unroll
                for (int q = 0; q < FG; ++q) {
                    const double zg = in ? ((double)grow[q][c0 + i] - gmu[q]) * gsc[q] : 0.0;
    #pragma unroll
                    for (int l = 0; l < FX; ++l) acc[q][l] = fma(zg, zf_[l], acc[q][l]);
                }
            }
        }
        double* Gt = G + (int64_t)t * mp * mp;
    #pragma unroll
        for (int q = 0; q < FG; ++q) {
    #pragma unroll
            for (int l = 0; l < FX; ++l) {
                double v = acc[q][l];
    #pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(L0S_FULL, v, o);
                const int64_t g = g0 + q;
                const int f = frow[l];
                if (lane == 0 && f >= 0 && g <= m) {
                    Gt[(int64_t)f * mp + g] = v;
                    Gt[g * mp + f] = v;
                }
            }
        }
    }  // batches
}

}  // namespace

int64_t ozaki_q_bytes(int64_t mp, int T, const int64_t* rpad_h, int64_t* KP_out) {
    const int64_t R = (mp + OZ_BM - 1) / OZ_BM * OZ_BM;
    int64_t KP = 0;
    for (int t = 0; t < T; ++t) KP += (rpad_h[t] + OZ_KC - 1) / OZ_KC * OZ_KC;
    if (KP_out) *KP_out = KP;
    return (int64_t)OZ_S * R * KP;
}

// Z (mp x sp, task t's columns [zoff_t, +rpad_t)) -> G (T x mp x mp) and eta (T); workspaces:
// Q (ozaki_q_bytes), ex (T x R ints), koff_d (T+1 int64, filled here).  Returns 0, or -1 when
// the TMA descriptor could not be built.
void ozaki_prepare_digits(int64_t m, int64_t mp, int T, const int64_t* rpad_h, int8_t* Q, int* ex, int64_t* koff_d,
                          DigitOut* out, cudaStream_t st, double* musc) {
    const int64_t R = (mp + OZ_BM - 1) / OZ_BM * OZ_BM;
    std::vector<int64_t> koff((size_t)T + 1, 0);
    for (int t = 0; t < T; ++t) koff[(size_t)t + 1] = koff[(size_t)t] + (rpad_h[t] + OZ_KC - 1) / OZ_KC * OZ_KC;
    const int64_t KP = koff[(size_t)T];
    cudaMemcpyAsync(koff_d, koff.data(), sizeof(int64_t) * (T + 1), cudaMemcpyHostToDevice, st);
    for (int a = 0; a < OZ_S; ++a) cudaMemsetAsync(Q + ((int64_t)a * R + m + 1) * KP, 0, (size_t)((R - m - 1) * KP), st);
    cudaMemsetAsync(ex, 0, sizeof(int) * T * R, st);
    *out = DigitOut{Q, R, KP, koff_d, ex};
    out->musc = musc;
}

static int oz_tiles_before(int gb) {  // tiles in column blocks [0, gb)
    int n = 0;
    for (int g = 0; g < gb; ++g) n += oz_tiles_in_block(g);
    return n;
}

// column blocks [0, upto) whose tiles only need rows < r1 (a landed row chunk completes them)
int ozaki_blocks_ready(int64_t r1) {
    int gb = 0;
    while ((int64_t)oz_tiles_in_block(gb) * OZ_BM <= r1) ++gb;
    return gb;
}

int ozaki_col_blocks(int64_t mp) { return (int)((mp + OZ_BM - 1) / OZ_BM * OZ_BM / OZ_BN); }

int launch_ozaki_tiles(int T, int64_t mp, const int64_t* rpad_h, const int8_t* Q, const int* ex,
                       const int64_t* koff_d, double* G, int gb0, int gb1, cudaStream_t st) {
    const int64_t R = (mp + OZ_BM - 1) / OZ_BM * OZ_BM;
    const int nbc = (int)(R / OZ_BN);
    gb1 = std::min(gb1, nbc);
    if (gb1 <= gb0) return 0;
    int64_t KP = 0;
    for (int t = 0; t < T; ++t) KP += (rpad_h[t] + OZ_KC - 1) / OZ_KC * OZ_KC;
    TmaDesc tmA, tmB;
    if (!make_tma_i8_3d(&tmA, Q, (unsigned long long)KP, (unsigned long long)R, OZ_S, OZ_KC, OZ_BM) ||
        !make_tma_i8_3d(&tmB, Q, (unsigned long long)KP, (unsigned long long)R, OZ_S, OZ_KC, OZ_BN))
        return -1;
    cudaFuncSetAttribute(k_oz_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    const int t0 = oz_tiles_before(gb0), t1 = oz_tiles_before(gb1);
    k_oz_gemm<<<dim3((unsigned)(t1 - t0), (unsigned)T), 192, OZ_SMEM, st>>>(tmA, tmB, koff_d, ex, R, nbc, mp, G, t0);
    return 0;
}

void launch_ozaki_eta(int T, int64_t m, int64_t mp, const int* ex, const double* rows_d, const double* G, double* eta_d,
                      cudaStream_t st, const OzFix* fix) {
    const int64_t R = (mp + OZ_BM - 1) / OZ_BM * OZ_BM;
    k_oz_eta<<<1, 1024, 0, st>>>(ex, R, T, m, mp, G, rows_d, OZ_ETA_MAX, eta_d, fix ? fix->rows : nullptr,
                                 fix ? fix->count : nullptr, fix ? fix->cap : 0, fix ? fix->flags : nullptr);
}

void launch_ozaki_fixup(const void* Xp, const void* yp, int precision, int64_t m, int64_t s, const int64_t* bounds_d,
                        int T, const double* musc, int64_t R, int64_t mp, const OzFix& fix, double* G, cudaStream_t st) {
    const int64_t per = (FTH / 32) * FG;
    const dim3 grid((unsigned)((m + 1 + per - 1) / per), (unsigned)T);
    if (precision == 1)
        k_oz_fixup<float><<<grid, FTH, 0, st>>>((const float*)Xp, (const float*)yp, m, s, bounds_d, musc, R, mp, fix.rows,
                                                fix.count, fix.cap, G);
    else
        k_oz_fixup<double><<<grid, FTH, 0, st>>>((const double*)Xp, (const double*)yp, m, s, bounds_d, musc, R, mp,
                                                 fix.rows, fix.count, fix.cap, G);
}

int launch_ozaki_gram(const double* Z, int64_t sp, const int64_t* zoff_d, const int64_t* rpad_h, int T, int64_t m,
                      int64_t mp, const double* rows_d, double* G, double* eta_d, int8_t* Q, int* ex, int64_t* koff_d,
                      bool digits_ready, cudaStream_t st, const OzFix* fix) {
    const int64_t R = (mp + OZ_BM - 1) / OZ_BM * OZ_BM;
    if (!digits_ready) {
        DigitOut dig;
        ozaki_prepare_digits(mp - 1, mp, T, rpad_h, Q, ex, koff_d, &dig, st);  // rows < mp come from Z here
        const int64_t warps = mp * T;
        k_oz_split<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(Z, sp, zoff_d, T, mp, R, koff_d, Q, dig.KP,
                                                                          ex);
    }
    if (launch_ozaki_tiles(T, mp, rpad_h, Q, ex, koff_d, G, 0, ozaki_col_blocks(mp), st)) return -1;
    launch_ozaki_eta(T, m, mp, ex, rows_d, G, eta_d, st, digits_ready ? fix : nullptr);
    return 0;
}

}  // namespace l0s
