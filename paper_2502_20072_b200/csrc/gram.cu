// gram.cu -- per-task normalized Gram  G_t = Z_t Z_t^T  on the FP64 tensor path.
//
// Z is (mp x sp) row-major, sample-contiguous; task t owns columns
// [zoff_t, zoff_t + rpad_t).  Row m of Z is the centered property, so the
// augmented Gram carries c_i = z_i . y_c in column m and |y_c|^2 at (m, m).
// One CTA computes one 64x64 block of the upper triangle (both triangles are
// written), streaming K in 32-sample chunks through a cp.async double buffer.
// Warp tile 16x32 = 2x4 m8n8 fragments; every k4 step issues 8
// mma.sync.m8n8k4.f64 (SASS: DMMA.8x8x4) from 6 conflict-free LDS.64.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {
constexpr int BM = 64;   // block edge
constexpr int BK = 32;   // k chunk (doubles)
constexpr int LDS = BK + 4;  // padded smem row (36 doubles = 288 B): rows 0..3 and 4..7 of a fragment hit disjoint banks

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Block (task, ba, bb), ba <= bb, of the linear index g over T x (upper-triangle blocks).
__device__ __forceinline__ void gram_block(int64_t g, int nb, int& task, int& ba, int& bb) {
    const int nblk = nb * (nb + 1) / 2;
    task = (int)(g / nblk);
    int lin = (int)(g % nblk);
    ba = 0;
    while (lin >= nb - ba) {
        lin -= nb - ba;
        ++ba;
    }
    bb = ba + lin;
}

// grid: blocks [g0, g0 + gridDim.x) of the linear (task, upper-triangle block) order; task t owns
// Z columns [zoff[t], zoff[t+1]) and G + t mp^2.  pack == nullptr: write G (both triangles);
// otherwise write block g - g0 as a row-major 64 x 64 tile at pack + (g - g0) * 4096 (a shard
// of the multi-GPU Gram, exchanged by all-gather and scattered by k_gram_unpack).
// colmajor != 0: blockIdx.y is the task and g0 + blockIdx.x indexes that task's upper-triangle
// blocks column by column (bb outer, ba = 0..bb inner), so a range of column block-rows is a
// contiguous range of blocks.
// NW warps (8: warp tile 16 x 32, 4: warp tile 32 x 32 with twice the accumulators per warp)
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_gram(const double* __restrict__ Z, int64_t sp,
                                                  const int64_t* __restrict__ zoff, int nb, double* __restrict__ Gall,
                                                  int64_t mp, int64_t g0, double* __restrict__ pack, int colmajor) {
    constexpr int FA = 64 / (NW / 2) / 8;  // row fragments per warp
    extern __shared__ __align__(16) double gsm[];
    double* sA[2] = {gsm, gsm + BM * LDS};
    double* sB[2] = {gsm + 2 * BM * LDS, gsm + 3 * BM * LDS};
    int task, ba, bb;
    if (colmajor) {
        task = blockIdx.y;
        const int64_t g = g0 + blockIdx.x;
        bb = (int)((sqrt(8.0 * (double)g + 1.0) - 1.0) * 0.5);
        while ((int64_t)(bb + 1) * (bb + 2) / 2 <= g) ++bb;
        while ((int64_t)bb * (bb + 1) / 2 > g) --bb;
        ba = (int)(g - (int64_t)bb * (bb + 1) / 2);
    } else {
        gram_block(g0 + blockIdx.x, nb, task, ba, bb);
    }
    const int64_t k0 = zoff[task], klen = zoff[task + 1] - k0;
    double* G = Gall + (int64_t)task * mp * mp;
    const double* Za = Z + (int64_t)ba * BM * sp + k0;
    const double* Zb = Z + (int64_t)bb * BM * sp + k0;
    int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int nchunks = (int)((klen + BK - 1) / BK);

    auto load = [&](int buf, int c) {
        int64_t kc = (int64_t)c * BK;
        int valid = (int)((klen - kc) < BK ? (klen - kc) : BK);  // multiple of 8
        // 64 rows x (valid/2) 16-byte pieces per operand
        int pieces = BM * (valid / 2);
        for (int p = tid; p < 2 * pieces; p += NW * 32) {
            int which = p >= pieces;
            int q = which ? p - pieces : p;
            int row = q / (valid / 2), col = (q % (valid / 2)) * 2;
            const double* src = (which ? Zb : Za) + (int64_t)row * sp + kc + col;
            double* dst = (which ? sB[buf] : sA[buf]) + row * LDS + col;
            cp_async16(dst, src);
        }
        cp_async_commit();
    };

    double acc[FA][4][2];
#pragma unroll
    for (int a = 0; a < FA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    int r0 = (warp >> 1) * (8 * FA), c0 = (warp & 1) * 32;
    int fr = lane >> 2, fk = lane & 3;
    load(0, 0);
    for (int c = 0; c < nchunks; ++c) {
        int buf = c & 1;
        if (c + 1 < nchunks) {
            load(buf ^ 1, c + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        int64_t kc = (int64_t)c * BK;
        int valid = (int)((klen - kc) < BK ? (klen - kc) : BK);
        const double* A = sA[buf];
        const double* B = sB[buf];
        for (int kk = 0; kk < valid; kk += 4) {
            double av[FA], b[4];
#pragma unroll
            for (int a = 0; a < FA; ++a) av[a] = A[(r0 + a * 8 + fr) * LDS + kk + fk];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = B[(c0 + j * 8 + fr) * LDS + kk + fk];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int a = 0; a < FA; ++a) dmma(acc[a][j][0], acc[a][j][1], av[a], b[j]);
        }
        __syncthreads();
    }
    // epilogue: fragment (row = lane/4, col = 2*(lane%4) + v)
    double* P = pack ? pack + (int64_t)blockIdx.x * (BM * BM) : nullptr;
#pragma unroll
    for (int a = 0; a < FA; ++a)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int lr = r0 + a * 8 + fr, lc = c0 + j * 8 + 2 * fk + v;
                const double x = acc[a][j][v];
                if (P) {
                    P[lr * BM + lc] = x;
                } else {
                    const int64_t row = (int64_t)ba * BM + lr, col = (int64_t)bb * BM + lc;
                    G[row * mp + col] = x;
                    if (ba != bb) G[col * mp + row] = x;
                }
            }
}

// Scatter all shards' packed tiles into G (both triangles; the mirror goes through shared
// memory so both stores are coalesced).  recv = nshards x per_shard tiles, shard r holding
// blocks [r * per_shard, ...) of the linear order, total blocks overall.
__global__ void __launch_bounds__(256) k_gram_unpack(const double* __restrict__ recv, int64_t total, int nb,
                                                     double* __restrict__ Gall, int64_t mp) {
    __shared__ double t[BM][BM + 1];
    const int64_t g = blockIdx.x;
    if (g >= total) return;
    int task, ba, bb;
    gram_block(g, nb, task, ba, bb);
    double* G = Gall + (int64_t)task * mp * mp;
    const double* P = recv + g * (BM * BM);
    for (int e = threadIdx.x; e < BM * BM; e += blockDim.x) {
        const int r = e / BM, c = e % BM;
        const double x = P[e];
        G[((int64_t)ba * BM + r) * mp + (int64_t)bb * BM + c] = x;
        t[r][c] = x;
    }
    if (ba == bb) return;
    __syncthreads();
    for (int e = threadIdx.x; e < BM * BM; e += blockDim.x) {
        const int r = e / BM, c = e % BM;
        G[((int64_t)bb * BM + r) * mp + (int64_t)ba * BM + c] = t[c][r];
    }
}

__global__ void k_unit_diag(double* Gall, int64_t m, int64_t mp) {
    int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double* G = Gall + (int64_t)blockIdx.y * mp * mp;
    if (f < m) {
        double d = G[f * mp + f];
        G[f * mp + f] = (d == d) ? 1.0 : d;  // keep NaN rows NaN (constant feature)
    }
}
__global__ void k_mark_dead(double* G, const int32_t* dead, int ndead, int T, int64_t mp) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)ndead * T * mp;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = e % mp;
        int t = (int)((e / mp) % T);
        int64_t f = dead[e / (mp * T)];
        double* Gt = G + (int64_t)t * mp * mp;
        Gt[f * mp + x] = nan;
        Gt[x * mp + f] = nan;
    }
}
}  // namespace

void launch_mark_dead(double* G, const int32_t* dead, int ndead, int T, int64_t mp, cudaStream_t st) {
    if (ndead > 0) k_mark_dead<<<256, 256, 0, st>>>(G, dead, ndead, T, mp);
}

static void gram_launch(dim3 grid, const double* Z, int64_t sp, const int64_t* zoff_d, int nb, double* G, int64_t mp,
                        int64_t g0, double* pack, int colmajor, cudaStream_t st) {
    static const int nw = [] {
        const char* e = getenv("L0S_GRAM_W");
        return (e && atoi(e) == 4) ? 4 : 8;
    }();
    const int smem = 4 * BM * LDS * (int)sizeof(double);
    if (nw == 4) {
        cudaFuncSetAttribute(k_gram<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_gram<4><<<grid, 128, smem, st>>>(Z, sp, zoff_d, nb, G, mp, g0, pack, colmajor);
    } else {
        cudaFuncSetAttribute(k_gram<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_gram<8><<<grid, 256, smem, st>>>(Z, sp, zoff_d, nb, G, mp, g0, pack, colmajor);
    }
}

int64_t gram_blocks(int64_t mp, int T) {
    const int64_t nb = mp / BM;
    return (int64_t)T * (nb * (nb + 1) / 2);
}
int64_t gram_shard_blocks(int64_t mp, int T, int nshards) {
    return (gram_blocks(mp, T) + nshards - 1) / nshards;
}

void launch_gram(const double* Z, int64_t sp, const int64_t* zoff_d, int T, int64_t mp, double* G, int shard,
                 int nshards, double* pack, cudaStream_t st) {
    const int nb = (int)(mp / BM);
    const int64_t total = gram_blocks(mp, T);
    // one launch for every task: ~T * nb^2 / 2 CTAs keep the tail wave short
    int64_t g0 = 0, cnt = total;
    if (nshards > 1) {
        const int64_t per = gram_shard_blocks(mp, T, nshards);
        g0 = std::min<int64_t>(total, per * shard);
        cnt = std::min<int64_t>(total, g0 + per) - g0;
    }
    if (cnt > 0) gram_launch(dim3((unsigned)cnt), Z, sp, zoff_d, nb, G, mp, g0, nshards > 1 ? pack : nullptr, 0, st);
}

void launch_gram_cols(const double* Z, int64_t sp, const int64_t* zoff_d, int T, int64_t mp, double* G, int B0,
                      int B1, cudaStream_t st) {
    const int nb = (int)(mp / BM);
    if (B1 > nb) B1 = nb;
    if (B1 <= B0) return;
    const int64_t g0 = (int64_t)B0 * (B0 + 1) / 2, g1 = (int64_t)B1 * (B1 + 1) / 2;
    gram_launch(dim3((unsigned)(g1 - g0), (unsigned)T), Z, sp, zoff_d, nb, G, mp, g0, nullptr, 1, st);
}

void launch_gram_unpack(const double* recv, int T, int64_t mp, double* G, cudaStream_t st) {
    const int64_t total = gram_blocks(mp, T);
    k_gram_unpack<<<(unsigned)total, 256, 0, st>>>(recv, total, (int)(mp / BM), G, mp);
}

void launch_unit_diag(double* G, int T, int64_t m, int64_t mp, cudaStream_t st) {
    k_unit_diag<<<dim3((unsigned)((m + 255) / 256), (unsigned)T), 256, 0, st>>>(G, m, mp);
}

}  // namespace l0s
