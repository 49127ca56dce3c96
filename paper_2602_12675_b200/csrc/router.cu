// router.cu -- the learnable router of SLA2 on sm_100a, bit-exact with the reference.
//
// Replaces (all file:line under /root/reference/proj/include/sla2):
//   colmean + smooth_k          matrix.hpp:235-244, quant.hpp:88-96
//   mean_pool (x2)              matrix.hpp:174-195
//   matmul (projections)        matrix.hpp:101-135 (i-k-j order), scale 272-277
//   block_scores                router.hpp:87-102
//   row_softmax                 matrix.hpp:138-155 (libm expf -> expf_glibc)
//   topk_budget / hard_topk     router.hpp:36-40, 106-125
// Every float op that feeds the mask is an explicit round-to-nearest intrinsic in the
// reference's serial order (no FMA contraction, no re-association), so the mask bits and
// the ascending kept-block index lists equal the reference's for the same inputs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
    return __bfloat162float(x);
}

// acc + float(x), rounded once: for bf16 the sm_100 mixed-precision add (FHADD.BF16) -- the
// bf16 -> f32 widening is exact, so the result equals __fadd_rn(acc, float(x)) bit for bit,
// without a separate convert between the shared-memory load and the add chain.
__device__ __forceinline__ float add_widen(float acc, float x) { return __fadd_rn(acc, x); }
__device__ __forceinline__ float add_widen(float acc, __nv_bfloat16 x) {
    asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"(*reinterpret_cast<const unsigned short*>(&x)));
    return acc;
}

// ---------------------------------------------------------------------------------------------
// K0: mu[bh][c] = colmean(K[bh]) with the reference's serial row order (matrix.hpp:235-244):
// out[c] += x(i, c) for i ascending, then out[c] *= float(1) / float(rows). One lane per column:
// the add chain is a latency floor of N dependent FADDs; loads are batched
// ahead of the chain so it runs at FADD latency.
// grid (ceil(d/32), B*H), block 32.
template <typename T>
__global__ void __launch_bounds__(32) colmean_exact_kernel(const T* __restrict__ k, float* __restrict__ mu, int N,
                                                           int d) {
    const int c = blockIdx.x * 32 + threadIdx.x;
    const int64_t bh = blockIdx.y;
    if (c >= d) return;
    const T* p = k + bh * (int64_t)N * d + c;
    float acc = 0.0f;
    constexpr int U = 32;
    int i = 0;
    for (; i + U <= N; i += U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = to_f32(p[(int64_t)(i + u) * d]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __fadd_rn(acc, v[u]);
    }
    for (; i < N; ++i) acc = __fadd_rn(acc, to_f32(p[(int64_t)i * d]));
    const float inv = __fdiv_rn(1.0f, (float)N);
    mu[bh * d + c] = __fmul_rn(acc, inv);
}

// K0, TMA-fed: one CTA per (group of 128-byte column strips, bh): 64 bf16 / 32 fp32 columns,
// so every TMA box row is a full 128-byte segment. The last warp streams [128 rows x COLS]
// tiles into an 8-deep shared-memory ring; each compute warp runs 32 serial add chains out of
// shared memory with register double-buffering, so each chain runs at FADD latency instead of
// DRAM latency. Same order and roundings as colmean_exact_kernel.
namespace cm {
constexpr int ROWS = 128, NST = 8;
}
#ifdef SLA2_TRACE
// trace build only: per-chunk %globaltimer stamps of CTA (0, 0)'s first consumer thread
__device__ unsigned long long* g_cm_trace = nullptr;
extern "C" void sla2_cm_trace_set(unsigned long long* p) { cudaMemcpyToSymbol(g_cm_trace, &p, sizeof(p)); }
#endif
template <typename T>
__global__ void __launch_bounds__(96) colmean_tma_kernel(const __grid_constant__ CUtensorMap tmK, float* __restrict__ mu,
                                                         int N, int d) {
    constexpr int COLS = 128 / sizeof(T);
    constexpr int NCW = COLS / 32;  // compute warps
    extern __shared__ __align__(128) uint8_t smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);  // [NST][ROWS][COLS]
    __shared__ uint64_t full[cm::NST], empty[cm::NST];
    const int cg = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunk = N / cm::ROWS;  // N % 128 == 0 is checked by the launcher
    if (threadIdx.x == 0) {
        for (int s = 0; s < cm::NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], COLS);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == NCW) {
        if (lane == 0) {
            tma_prefetch_desc(&tmK);
            for (int c = 0; c < nchunk; ++c) {
                const int s = c % cm::NST;
                if (c >= cm::NST) mbar_wait(&empty[s], ((c / cm::NST) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], cm::ROWS * COLS * sizeof(T));
                tma_load_2d(ring + (size_t)s * cm::ROWS * COLS, &tmK, cg * COLS,
                            (int)(bh * N + (int64_t)c * cm::ROWS), &full[s]);
            }
        }
        return;
    }
    if (warp > NCW) return;
    const int col = warp * 32 + lane;
    float acc = 0.0f;
    // The FADD chain (4 cycles per row) is the floor; every other instruction must hide
    // under it. Rolling window: the load + convert of row r + W is issued right after the
    // FADD of row r, so each FADD has two independent instructions beside it. The window
    // runs across chunk boundaries (the next stage is waited for W rows early).
    constexpr int W = 16;
    T x[W];  // raw elements: the add widens them (add_widen)
    {
        mbar_wait(&full[0], 0);
        const T* tile = ring + col;
#pragma unroll
        for (int u = 0; u < W; ++u) x[u] = tile[u * COLS];
    }
    for (int c = 0; c < nchunk; ++c) {
        const int s = c % cm::NST;
        const T* tile = ring + (size_t)s * cm::ROWS * COLS + col;
#pragma unroll
        for (int r = 0; r < cm::ROWS - W; r += W) {
#pragma unroll
            for (int u = 0; u < W; ++u) {
                acc = add_widen(acc, x[u]);
                x[u] = tile[(r + W + u) * COLS];
            }
        }
        // last W rows of this chunk; prefetch the first W of the next
        const bool more = c + 1 < nchunk;
        const int s1 = (c + 1) % cm::NST;
        if (more) mbar_wait(&full[s1], ((c + 1) / cm::NST) & 1);
#ifdef SLA2_TRACE
        if (g_cm_trace && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && c < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            g_cm_trace[c] = t;
        }
#endif
        const T* nt = ring + (size_t)s1 * cm::ROWS * COLS + col;
#pragma unroll
        for (int u = 0; u < W; ++u) {
            acc = add_widen(acc, x[u]);
            if (more) x[u] = nt[u * COLS];
        }
        __syncwarp();
        mbar_arrive(&empty[s]);
    }
    const float inv = __fdiv_rn(1.0f, (float)N);
    mu[bh * d + cg * COLS + col] = __fmul_rn(acc, inv);
}

// K0 for bf16, transposed staging. The one-column-per-thread chain above loads one element per
// row (LDS.U16 -> FHADD): measured 7.4 cycles per row against the 4.5-cycle FADD latency
// (profiles/lat_bench_r01.txt), the per-load scoreboard wait being the difference. Here two
// transposer warps turn each TMA tile [128 rows][64 cols] into [64 cols][128 rows] (8x8 blocks:
// 8 x LDS.128, 32 PRMT, 8 x STS.128), so a chain thread gets 8 consecutive rows of its column
// from one LDS.128 and runs 8 FHADDs on registers. Same serial order, same bits.
// Transposed row of column c: 16 chunks of 8 rows, chunk rc at ((rc ^ key(c)) * 16): the XOR
// key spreads both the transposer's stores and the chain threads' loads over all banks.
namespace cmt {
constexpr int ROWS = 128, COLS = 64, NST = 8, NTS = 4;
constexpr int TILE = ROWS * COLS * 2;  // 16 KB (both layouts)
__device__ __forceinline__ uint32_t tpos(int c, int rc) {
    return (uint32_t)c * 256u + (uint32_t)((rc ^ ((c ^ (c >> 3)) & 7)) * 16);
}
}  // namespace cmt

__device__ __forceinline__ float add2_bf16(float acc, uint32_t w) {
    // acc + row(lo) then + row(hi): two FHADD.BF16, each rounded once (= fp32 add of the widened value)
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\t"
        "add.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %0, hi, %0;\n\t}"
        : "+f"(acc)
        : "r"(w));
    return acc;
}

__global__ void __launch_bounds__(160) colmean_tr_kernel(const __grid_constant__ CUtensorMap tmK, float* __restrict__ mu,
                                                         int N, int d) {
    using namespace cmt;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* ring = smem_raw;                   // [NST][128 rows][128 B]  (TMA)
    uint8_t* tring = smem_raw + NST * TILE;     // [NTS][64 cols][256 B]   (transposed)
    __shared__ uint64_t full[NST], empty[NST], tfull[NTS], tempty[NTS];
    const int cg = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5;
    const int nchunk = (N + ROWS - 1) / ROWS;  // rows past N (ragged tail) arrive as zeros
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 64);
        }
        for (int s = 0; s < NTS; ++s) {
            mbar_init(&tfull[s], 64);
            mbar_init(&tempty[s], 64);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 4) {  // TMA producer
        if ((threadIdx.x & 31) == 0) {
            tma_prefetch_desc(&tmK);
            for (int c = 0; c < nchunk; ++c) {
                const int s = c % NST;
                if (c >= NST) mbar_wait(&empty[s], ((c / NST) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], TILE);
                tma_load_3d(ring + s * TILE, &tmK, cg * COLS, c * ROWS, (int)bh, &full[s]);
            }
        }
        return;
    }
    // warps 0-1 transpose, 2-3 run the chains: each chain warp has an SM sub-partition (warp
    // scheduler) to itself; the TMA warp 4 shares scheduler 0 with a transposer
    if (warp < 2) {  // transposers: thread t owns 8x8 blocks (rb, cb) = (t/8 + 8k, t%8), k = 0, 1
        const int t = threadIdx.x;
        const int cb = t & 7;
        for (int c = 0; c < nchunk; ++c) {
            const int s = c % NST, ts = c % NTS;
            mbar_wait(&full[s], (c / NST) & 1);
            if (c >= NTS) mbar_wait(&tempty[ts], ((c / NTS) - 1) & 1);
            const uint32_t src = smem_u32(ring + s * TILE), dst = smem_u32(tring + ts * TILE);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int rb = (t >> 3) + 8 * k;
                uint32_t w[8][4];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    ld_shared_v4(src + (rb * 8 + i) * 128 + cb * 16, w[i][0], w[i][1], w[i][2], w[i][3]);
#pragma unroll
                for (int a = 0; a < 4; ++a) {  // columns 2a, 2a+1
                    uint32_t lo[4], hi[4];
#pragma unroll
                    for (int b = 0; b < 4; ++b) {  // rows 2b, 2b+1
                        lo[b] = __byte_perm(w[2 * b][a], w[2 * b + 1][a], 0x5410);
                        hi[b] = __byte_perm(w[2 * b][a], w[2 * b + 1][a], 0x7632);
                    }
                    const int c0 = cb * 8 + 2 * a;
                    st_shared_v4(dst + cmt::tpos(c0, rb), lo[0], lo[1], lo[2], lo[3]);
                    st_shared_v4(dst + cmt::tpos(c0 + 1, rb), hi[0], hi[1], hi[2], hi[3]);
                }
            }
            mbar_arrive(&empty[s]);
            mbar_arrive(&tfull[ts]);
        }
        return;
    }
    // chain threads: column col, 8 rows per LDS.128. Loads run two groups (16 rows, ~72 cycles
    // of adds) ahead of the chain, across chunk boundaries, so no add waits on shared memory.
    const int col = threadIdx.x - 64;
    float acc = 0.0f;
    uint32_t g0[4], g1[4];
    mbar_wait(&tfull[0], 0);
    {
        const uint32_t b0 = smem_u32(tring);
        ld_shared_v4(b0 + cmt::tpos(col, 0), g0[0], g0[1], g0[2], g0[3]);
        ld_shared_v4(b0 + cmt::tpos(col, 1), g1[0], g1[1], g1[2], g1[3]);
    }
    for (int c = 0; c < nchunk; ++c) {
        const int ts = c % NTS;
        const uint32_t base = smem_u32(tring + ts * TILE);
        const bool more = c + 1 < nchunk;
        const uint32_t nbase = smem_u32(tring + ((c + 1) % NTS) * TILE);
#pragma unroll
        for (int rc = 0; rc < 16; ++rc) {
            uint32_t g2[4] = {0u, 0u, 0u, 0u};
            if (rc + 2 < 16) {
                ld_shared_v4(base + cmt::tpos(col, rc + 2), g2[0], g2[1], g2[2], g2[3]);
            } else if (more) {
                if (rc == 14) mbar_wait(&tfull[(c + 1) % NTS], ((c + 1) / NTS) & 1);
                ld_shared_v4(nbase + cmt::tpos(col, rc - 14), g2[0], g2[1], g2[2], g2[3]);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) acc = add2_bf16(acc, g0[e]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                g0[e] = g1[e];
                g1[e] = g2[e];
            }
        }
        mbar_arrive(&tempty[ts]);
    }
    const float inv = __fdiv_rn(1.0f, (float)N);
    mu[bh * d + cg * COLS + col] = __fmul_rn(acc, inv);
}

// K0 (fast variant, exact_mu = 0): column sums in double over row chunks, then the same
// final scaling. Not the reference's order: the mask can differ at fp32 ties.
template <typename T>
__global__ void colmean_partial_kernel(const T* __restrict__ k, double* __restrict__ part, int N, int d,
                                       int rows_per_chunk) {
    const int c = threadIdx.x;
    const int64_t bh = blockIdx.y;
    const int chunk = blockIdx.x;
    const int r0 = chunk * rows_per_chunk;
    const int r1 = min(N, r0 + rows_per_chunk);
    double acc = 0.0;
    for (int r = r0; r < r1; ++r) acc += (double)to_f32(k[(bh * N + r) * (int64_t)d + c]);
    part[(bh * gridDim.x + chunk) * d + c] = acc;
}
__global__ void colmean_finish_kernel(const double* __restrict__ part, float* __restrict__ mu, int nchunks, int N,
                                      int d) {
    const int c = threadIdx.x;
    const int64_t bh = blockIdx.x;
    double acc = 0.0;
    for (int i = 0; i < nchunks; ++i) acc += part[(bh * nchunks + i) * d + c];
    const float inv = __fdiv_rn(1.0f, (float)N);
    mu[bh * d + c] = __fmul_rn(__double2float_rn(acc), inv);
}

// ---------------------------------------------------------------------------------------------
// K1a/K1b: pooled + projected blocks.
//   xbar[g][c] = float( (sum_r (double)x~[g*b + r][c]) / (double)b )     (matrix.hpp:180-192)
//   xp[g][c]   = sum_f xbar[g][f] * P[f][c], f ascending, from 0          (matrix.hpp:121-132)
// with x~ = fl(K - mu) for keys when smoothing (quant.hpp:93), x for queries.
// grid (nblocks, B*H), block d. Dynamic smem: d floats.
template <typename T>
__global__ void pool_project_kernel(const T* __restrict__ x, const float* __restrict__ mu, const float* __restrict__ proj,
                                    float* __restrict__ xp, int N, int d, int H, int block,
                                    float* __restrict__ xbar_out, __nv_bfloat16* __restrict__ phi_out) {
    extern __shared__ __align__(16) uint8_t psm[];
    float* sbar = reinterpret_cast<float*>(psm);
    T* tile = reinterpret_cast<T*>(psm + ((d * sizeof(float) + 15) & ~size_t(15)));  // [block][d]
    const int c = threadIdx.x;
    const int g = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int h = (int)(bh % H);
    const int nblk = (N + block - 1) / block;
    const int cnt = min(block, N - g * block);  // rows of this block (ragged tail: fewer)
    // stage the whole [cnt x d] slab with independent 16-byte loads (one DRAM round trip)
    {
        const T* src = x + (bh * N + (int64_t)g * block) * d;
        if (((d * sizeof(T)) & 15) == 0) {
            const int n16 = (int)((size_t)cnt * d * sizeof(T) / 16);
            stage_copy<16>(reinterpret_cast<uint4*>(tile), reinterpret_cast<const uint4*>(src), n16, c, blockDim.x);
        } else {
            for (int e = c; e < cnt * d; e += blockDim.x) tile[e] = src[e];
        }
    }
    __syncthreads();
    if (phi_out) {
        // phi(Q) rows from the staged tile (bf16, d = 128): phiq_kernel's arithmetic (16 lanes
        // per row, 8 features each), so Q is read from DRAM once for pooling and phi(Q)
        const int sub = c & 15, rpp = (int)(blockDim.x >> 4);  // rows per pass
        for (int r0 = 0; r0 < cnt; r0 += rpp) {  // every lane runs every pass (shuffles)
            const int r = r0 + (c >> 4);
            const bool live = r < cnt;
            const int rr = live ? r : cnt - 1;
            const uint4 w = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(tile) + rr * 128 + sub * 8);
            const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
            float xv[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
                xv[2 * e] = f2.x;
                xv[2 * e + 1] = f2.y;
            }
            float mx = fmaxf(fmaxf(fmaxf(xv[0], xv[1]), fmaxf(xv[2], xv[3])), fmaxf(fmaxf(xv[4], xv[5]), fmaxf(xv[6], xv[7])));
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float sum = 0.0f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                float y;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"((xv[e] - mx) * 1.4426950408889634f));
                xv[e] = y;
                sum += y;
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const float inv = 1.0f / sum;
            uint4 o4;
            o4.x = pack_bf16(xv[0] * inv, xv[1] * inv);
            o4.y = pack_bf16(xv[2] * inv, xv[3] * inv);
            o4.z = pack_bf16(xv[4] * inv, xv[5] * inv);
            o4.w = pack_bf16(xv[6] * inv, xv[7] * inv);
            if (live) *reinterpret_cast<uint4*>(phi_out + (bh * N + (int64_t)g * block + r) * 128 + sub * 8) = o4;
        }
    }
    const float m = mu ? mu[bh * d + c] : 0.0f;
    double acc = 0.0;
    for (int r = 0; r < cnt; ++r) {
        float v = to_f32(tile[r * d + c]);
        if (mu) v = __fsub_rn(v, m);
        acc = __dadd_rn(acc, (double)v);
    }
    sbar[c] = __double2float_rn(__ddiv_rn(acc, (double)cnt));
    if (xbar_out) {  // pooled rows only; the projection runs in project_kernel
        xbar_out[(bh * nblk + g) * d + c] = sbar[c];
        return;
    }
    __syncthreads();
    const float* P = proj + (int64_t)h * d * d;
    float o = 0.0f;
    int f = 0;
    for (; f + 16 <= d; f += 16) {
        float pv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) pv[u] = P[(int64_t)(f + u) * d + c];
#pragma unroll
        for (int u = 0; u < 16; ++u) o = __fadd_rn(o, __fmul_rn(sbar[f + u], pv[u]));
    }
    for (; f < d; ++f) o = __fadd_rn(o, __fmul_rn(sbar[f], P[(int64_t)f * d + c]));
    xp[(bh * nblk + g) * d + c] = o;
}

// xp[g][c] = sum_f xbar[g][f] * P[f][c] (matrix.hpp:121-132: i-k-j order, one serial chain
// per output, f ascending from 0, separate mul and add), for a tile of 32 pooled rows x cw
// output columns per CTA (cw = 64, or d, or 16: a divisor of d): P[:, tile] and the xbar rows live in shared memory;
// each of the 2 cw threads owns a 4 x 4 register tile of outputs (16 independent chains) and
// steps f by 4 with vector loads. grid (ceil(nrows/32), d/cw, BH), block 2 cw. Requires
// d % 16 == 0. The column split keeps ~4 CTAs per SM (the kernel is latency-bound at low
// occupancy). With xp_t the output is written transposed, [BH][d][nrows]
// (the router's key side: lanes of router_rows_kernel then read consecutive keys of one
// feature, coalesced).
__global__ void __launch_bounds__(128) project_kernel(const float* __restrict__ xbar, const float* __restrict__ proj,
                                                      float* __restrict__ xp, int nrows, int d, int H, int xp_t) {
    extern __shared__ __align__(16) float psh[];
    const int cw = blockDim.x / 2;
    float* sP = psh;            // [d][cw]
    float* sX = psh + d * cw;   // [32][d]
    const int64_t bh = blockIdx.z;
    const int h = (int)(bh % H);
    const int r0 = blockIdx.x * 32;
    const int c0 = blockIdx.y * cw;
    const int tid = threadIdx.x;
    const int nr = min(32, nrows - r0);
    {
        // all of this CTA's loads in flight at once (a load / store loop would make one DRAM
        // round trip per iteration)
        const float* Pb = proj + (int64_t)h * d * d + c0;
        const int cw4 = cw / 4, np = d * cw4, nx = nr * d / 4;
        for (int base = tid; base < np; base += 16 * blockDim.x) {
            float4 t[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int e = base + u * blockDim.x;
                if (e < np) t[u] = *reinterpret_cast<const float4*>(Pb + (int64_t)(e / cw4) * d + (e % cw4) * 4);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int e = base + u * blockDim.x;
                if (e < np) reinterpret_cast<float4*>(sP)[e] = t[u];
            }
        }
        float4* x4 = reinterpret_cast<float4*>(sX);
        stage_copy<8>(x4, reinterpret_cast<const float4*>(xbar + (bh * nrows + r0) * (int64_t)d), nx, tid, blockDim.x);
        for (int e = nx + tid; e < 32 * d / 4; e += blockDim.x) x4[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const int ncg = cw / 4;
    const int cg = tid % ncg, rg = tid / ncg;  // 8 row groups of 4 rows
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
    for (int f = 0; f < d; f += 4) {
        float4 pv[4], xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = *reinterpret_cast<const float4*>(sP + (f + u) * cw + cg * 4);
#pragma unroll
        for (int a = 0; a < 4; ++a) xv[a] = *reinterpret_cast<const float4*>(sX + (rg * 4 + a) * d + f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const float x = u == 0 ? xv[a].x : u == 1 ? xv[a].y : u == 2 ? xv[a].z : xv[a].w;
                const float2 x2 = make_float2(x, x);  // packed FMUL2 products, scalar FADD sums
                const float2 p01 = __fmul2_rn(x2, make_float2(pv[u].x, pv[u].y));
                const float2 p23 = __fmul2_rn(x2, make_float2(pv[u].z, pv[u].w));
                acc[a][0] = __fadd_rn(acc[a][0], p01.x);
                acc[a][1] = __fadd_rn(acc[a][1], p01.y);
                acc[a][2] = __fadd_rn(acc[a][2], p23.x);
                acc[a][3] = __fadd_rn(acc[a][3], p23.y);
            }
        }
    }
    const int col = c0 + cg * 4;
    if (xp_t) {
        // transposed rows padded to a multiple of 4 keys (aligned float4 rows for any tn)
        const int ldt = (nrows + 3) & ~3;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            float* dst = xp + (bh * d + col + b) * (int64_t)ldt + r0 + rg * 4;
            if (rg * 4 + 4 <= nr) {
                *reinterpret_cast<float4*>(dst) = make_float4(acc[0][b], acc[1][b], acc[2][b], acc[3][b]);
            } else {
#pragma unroll
                for (int a = 0; a < 4; ++a)
                    if (rg * 4 + a < nr) dst[a] = acc[a][b];
            }
        }
    } else {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int r = rg * 4 + a;
            if (r < nr)
                *reinterpret_cast<float4*>(xp + (bh * nrows + r0 + r) * (int64_t)d + col) =
                    make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
        }
    }
}

static void launch_project(const float* xbar, const float* proj, float* xp, int nrows, int d, int H, int BH, int xp_t,
                           cudaStream_t st) {
    const int cw = d % 64 == 0 ? 64 : (d <= 64 ? d : 16);  // a divisor of d (d % 16 == 0)
    const size_t ps = ((size_t)d * cw + 32 * (size_t)d) * 4;
    if (ps > 48 * 1024) cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    project_kernel<<<dim3((nrows + 31) / 32, d / cw, BH), 2 * cw, ps, st>>>(xbar, proj, xp, nrows, d, H, xp_t);
}

// ---------------------------------------------------------------------------------------------
// Top-k over one row held in shared memory (router.hpp:106-125). Keys sort by (value desc,
// column asc) -- exactly std::stable_sort with `pc(i,a) > pc(i,b)`. Equal values (incl. -0/+0)
// tie and the lower column wins. Writes mask bits (tn) and the kept columns ascending (kappa).
__device__ __forceinline__ uint32_t desc_key(float v) {
    uint32_t u = __float_as_uint(v);
    if (u == 0x80000000u) u = 0;  // -0 == +0
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // ascending float order as unsigned
    return ~u;                                         // descending
}

__device__ void topk_row(const float* __restrict__ vals, int tn, int kappa, unsigned long long* keys, int npow2,
                         uint8_t* __restrict__ mask_row, int32_t* __restrict__ idx_row, uint8_t* sel, int* warp_cnt) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int j = tid; j < npow2; j += nt)
        keys[j] = (j < tn) ? (((unsigned long long)desc_key(vals[j]) << 32) | (unsigned)j) : ~0ull;
    __syncthreads();
    // bitonic sort ascending
    for (int size = 2; size <= npow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < npow2 / 2; t += nt) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < tn; j += nt) sel[j] = 0;
    __syncthreads();
    for (int r = tid; r < kappa; r += nt) sel[(int)(keys[r] & 0xffffffffu)] = 1;
    __syncthreads();
    if (mask_row)
        for (int j = tid; j < tn; j += nt) mask_row[j] = sel[j];
    // ascending compaction of the kept columns
    const int nwarps = (nt + 31) >> 5;
    int base = 0;
    for (int j0 = 0; j0 < tn; j0 += nt) {
        const int j = j0 + tid;
        const bool f = (j < tn) && sel[j];
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if ((tid & 31) == 0) warp_cnt[tid >> 5] = __popc(bal);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < (tid >> 5); ++w) before += warp_cnt[w];
        const int pos = base + before + __popc(bal & ((1u << (tid & 31)) - 1u));
        if (f && idx_row) idx_row[pos] = j;
        int tot = 0;
        for (int w = 0; w < nwarps; ++w) tot += warp_cnt[w];
        __syncthreads();
        base += tot;
    }
}

// K1d: one CTA per (bh, query block i):
//   s[j]  = (sum_c qp[i][c] * kp[j][c], c ascending, from 0) * inv_sqrt_d    (matrix.hpp:111-118,
//                                                                           router.hpp:99-100)
//   pc[j] = row_softmax(s)[j]: m = max, e = expf(s - m), serial sum over j ascending,
//           inv = 1/sum, pc = e * inv                                       (matrix.hpp:144-152)
// then hard top-kappa. Dynamic smem: tn floats (vals) + npow2 u64 keys + tn bytes + d floats.
__global__ void router_scores_topk_kernel(const float* __restrict__ qp, const float* __restrict__ kp,
                                          float inv_sqrt_d, int tm, int tn, int d, int kappa, int npow2,
                                          float* __restrict__ pc_out, uint8_t* __restrict__ mask_out,
                                          int32_t* __restrict__ idx_out) {
    extern __shared__ __align__(16) uint8_t smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    float* vals = reinterpret_cast<float*>(keys + npow2);
    float* sq = vals + tn;
    uint8_t* sel = reinterpret_cast<uint8_t*>(sq + d);
    __shared__ float red[32];
    __shared__ int warp_cnt[32];
    __shared__ float s_sum;
    const int i = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int c = tid; c < d; c += nt) sq[c] = qp[(bh * tm + i) * d + c];
    __syncthreads();
    const float* kpb = kp + bh * (int64_t)tn * d;
    float lmax = -INFINITY;
    for (int j = tid; j < tn; j += nt) {
        float acc = 0.0f;
        if ((d & 3) == 0) {
            const float4* kr = reinterpret_cast<const float4*>(kpb + (int64_t)j * d);
            for (int c4 = 0; c4 < d / 4; ++c4) {
                const float4 kv = kr[c4];
                acc = __fadd_rn(acc, __fmul_rn(sq[4 * c4 + 0], kv.x));
                acc = __fadd_rn(acc, __fmul_rn(sq[4 * c4 + 1], kv.y));
                acc = __fadd_rn(acc, __fmul_rn(sq[4 * c4 + 2], kv.z));
                acc = __fadd_rn(acc, __fmul_rn(sq[4 * c4 + 3], kv.w));
            }
        } else {
            for (int c = 0; c < d; ++c) acc = __fadd_rn(acc, __fmul_rn(sq[c], kpb[(int64_t)j * d + c]));
        }
        const float s = __fmul_rn(acc, inv_sqrt_d);
        vals[j] = s;
        lmax = fmaxf(lmax, s);
    }
    // block max (order-free)
    for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if ((tid & 31) == 0) red[tid >> 5] = lmax;
    __syncthreads();
    float m = red[0];
    for (int w = 1; w < (nt + 31) / 32; ++w) m = fmaxf(m, red[w]);
    for (int j = tid; j < tn; j += nt) vals[j] = expf_glibc(__fsub_rn(vals[j], m));
    __syncthreads();
    if (tid == 0) {  // serial sum, j ascending (matrix.hpp:148-149)
        float sum = 0.0f;
        for (int j = 0; j < tn; ++j) sum = __fadd_rn(sum, vals[j]);
        s_sum = __fdiv_rn(1.0f, sum);
    }
    __syncthreads();
    const float inv = s_sum;
    for (int j = tid; j < tn; j += nt) {
        const float p = __fmul_rn(vals[j], inv);
        vals[j] = p;
        if (pc_out) pc_out[(bh * tm + i) * (int64_t)tn + j] = p;
    }
    __syncthreads();
    topk_row(vals, tn, kappa, keys, npow2, mask_out ? mask_out + (bh * tm + i) * (int64_t)tn : nullptr,
             idx_out + (bh * tm + i) * (int64_t)kappa, sel, warp_cnt);
}

// Warp-local top-k, one warp per row, tn <= 32 * TKMAX keys (lane l holds j = l + 32u), any
// kappa <= tn: a radix select on the 32-bit descending keys finds T, the kappa-th best value
// (32 rounds of one compare per key and a warp add), then every key better than T is kept and
// the ties at T in ascending column order -- exactly std::stable_sort with pc(i,a) > pc(i,b)
// (router.hpp:117-122). About 2 * 32 * TKMAX instructions per row, against kappa rescans of
// TKMAX 64-bit keys for a kappa-round argmax.
template <int TKMAX>  // keys per lane: tn <= 32 * TKMAX
__device__ void warp_topk_small(float* __restrict__ vals, int tn, int kappa, uint8_t* __restrict__ mask_row,
                                int32_t* __restrict__ idx_row, uint8_t* sel) {
    const int lane = threadIdx.x & 31;
    // the row's keys replace its (already stored) probabilities in shared memory: no per-lane
    // key array, so a 2048-key row does not cost the kernel 64 registers (occupancy)
    uint32_t* hk = reinterpret_cast<uint32_t*>(vals);  // desc_key: smaller is better
    for (int j = lane; j < tn; j += 32) hk[j] = desc_key(vals[j]);
    __syncwarp();
    auto count_below = [&](uint32_t t) {
        int c = 0;
#pragma unroll 4
        for (int j = lane; j < tn; j += 32) c += hk[j] < t ? 1 : 0;
        return (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
    };
    // invariant: #(keys < prefix) < kappa
    uint32_t prefix = 0;
    for (int b = 31; b >= 0; --b) {
        const uint32_t cand = prefix | (1u << b);
        if (count_below(cand) < kappa) prefix = cand;
    }
    const int ties = kappa - count_below(prefix);  // keys equal to T = prefix still to keep
    const unsigned lt_mask = (1u << lane) - 1u;
    int taken = 0;
    for (int j0 = 0; j0 < tn; j0 += 32) {  // ascending columns: ties are kept lowest column first
        const int j = j0 + lane;
        const bool valid = j < tn;
        const uint32_t kj = valid ? hk[j] : 0xffffffffu;
        const bool eq = valid && kj == prefix;
        const unsigned eqm = __ballot_sync(0xffffffffu, eq);
        const bool take = valid && (kj < prefix || (eq && taken + __popc(eqm & lt_mask) < ties));
        taken += __popc(eqm);
        if (valid) sel[j] = take ? 1 : 0;
    }
    __syncwarp();
    int base = 0;
    for (int j0 = 0; j0 < tn; j0 += 32) {
        const int j = j0 + lane;
        const bool f = (j < tn) && sel[j];
        if (mask_row && j < tn) mask_row[j] = f ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) idx_row[base + __popc(bal & ((1u << lane) - 1u))] = j;
        base += __popc(bal);
    }
}

// Top-k by candidate bound (same result as warp_topk_small, ~4-7x fewer instructions):
//  1. each lane keeps its M smallest keys (32 M >= kappa); B = the kappa-th smallest of those
//     32 M values (radix select over them). At least kappa keys are <= B, so the kept set is
//     inside C = {j : key_j <= B} (ties at B included).
//  2. C is compacted in column order into `cand` as (key << 32 | column); if |C| > 64 the row
//     falls back to the full radix select.
//  3. a candidate is kept iff fewer than kappa candidates precede it in (key, column) order --
//     std::stable_sort's order (router.hpp:117-121).
template <int M>
__device__ void warp_topk_cand(float* __restrict__ vals, int tn, int kappa, uint8_t* __restrict__ mask_row,
                               int32_t* __restrict__ idx_row, uint8_t* sel, unsigned long long* cand) {
    const int lane = threadIdx.x & 31;
    uint32_t* hk = reinterpret_cast<uint32_t*>(vals);
    uint32_t lm[M];
#pragma unroll
    for (int t = 0; t < M; ++t) lm[t] = 0xffffffffu;
    for (int j = lane; j < tn; j += 32) {
        uint32_t k = desc_key(vals[j]);
        hk[j] = k;
#pragma unroll
        for (int t = 0; t < M; ++t) {  // insert into the lane's sorted M smallest
            const uint32_t lo = min(lm[t], k);
            k = max(lm[t], k);
            lm[t] = lo;
        }
    }
    __syncwarp();
    // B: kappa-th smallest of the 32 M lane minima (radix select; sentinels count as keys, so B
    // can only move up, never below the true kappa-th key)
    uint32_t prefix = 0;
    for (int b = 31; b >= 0; --b) {
        const uint32_t c = prefix | (1u << b);
        int n = 0;
#pragma unroll
        for (int t = 0; t < M; ++t) n += lm[t] < c ? 1 : 0;
        if ((int)__reduce_add_sync(0xffffffffu, (unsigned)n) < kappa) prefix = c;
    }
    const uint32_t B = prefix;
    // compact C in column order
    int base = 0;
    bool overflow = false;
    for (int j0 = 0; j0 < tn; j0 += 32) {
        const int j = j0 + lane;
        const uint32_t k = j < tn ? hk[j] : 0xffffffffu;
        const bool in = j < tn && k <= B;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        const int pos = base + __popc(bal & ((1u << lane) - 1u));
        if (in && pos < 64) cand[pos] = ((unsigned long long)k << 32) | (unsigned)j;
        base += __popc(bal);
    }
    overflow = base > 64;
    if (overflow) {  // uncommon: many keys tie near B; the exact radix select over the row
        __syncwarp();
        // warp_topk_small recomputes the keys from vals: restore the probabilities' order
        // encoding is monotone, so select on the keys already in hk
        uint32_t pfx = 0;
        auto count_below = [&](uint32_t t) {
            int c = 0;
            for (int j = lane; j < tn; j += 32) c += hk[j] < t ? 1 : 0;
            return (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
        };
        for (int b = 31; b >= 0; --b) {
            const uint32_t c = pfx | (1u << b);
            if (count_below(c) < kappa) pfx = c;
        }
        const int ties = kappa - count_below(pfx);
        const unsigned lt = (1u << lane) - 1u;
        int taken = 0;
        for (int j0 = 0; j0 < tn; j0 += 32) {
            const int j = j0 + lane;
            const bool valid = j < tn;
            const uint32_t kj = valid ? hk[j] : 0xffffffffu;
            const bool eq = valid && kj == pfx;
            const unsigned eqm = __ballot_sync(0xffffffffu, eq);
            const bool take = valid && (kj < pfx || (eq && taken + __popc(eqm & lt) < ties));
            taken += __popc(eqm);
            if (valid) sel[j] = take ? 1 : 0;
        }
    } else {
        for (int j = lane; j < tn; j += 32) sel[j] = 0;
        __syncwarp();
        // rank each candidate (lanes own candidates lane, lane + 32)
        for (int c = lane; c < base; c += 32) {
            const unsigned long long me = cand[c];
            int rank = 0;
            for (int e = 0; e < base; ++e) rank += cand[e] < me ? 1 : 0;
            if (rank < kappa) sel[(int)(me & 0xffffffffu)] = 1;
        }
    }
    __syncwarp();
    int ob = 0;
    for (int j0 = 0; j0 < tn; j0 += 32) {
        const int j = j0 + lane;
        const bool f = (j < tn) && sel[j];
        if (mask_row && j < tn) mask_row[j] = f ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) idx_row[ob + __popc(bal & ((1u << lane) - 1u))] = j;
        ob += __popc(bal);
    }
}

// Warp-local top-k on one row held in shared memory as 64-bit keys (value desc, column asc).
// Bitonic sort by one warp (npow2 / 64 compare-exchanges per lane per stage), then the kept
// columns are flagged and compacted in ascending order with ballots.
__device__ void warp_topk_row(const float* __restrict__ vals, int tn, int kappa, unsigned long long* keys,
                              int npow2, uint8_t* __restrict__ mask_row, int32_t* __restrict__ idx_row) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < npow2; j += 32)
        keys[j] = (j < tn) ? (((unsigned long long)desc_key(vals[j]) << 32) | (unsigned)j) : ~0ull;
    __syncwarp();
    for (int size = 2; size <= npow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < npow2 / 2; t += 32) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncwarp();
        }
    }
    // keys[0..kappa) are the kept columns; turn them into flags (reuse keys' tail as bytes)
    uint8_t* sel = reinterpret_cast<uint8_t*>(keys + npow2) ;  // caller reserves tn bytes after keys
    for (int j = lane; j < tn; j += 32) sel[j] = 0;
    __syncwarp();
    for (int r = lane; r < kappa; r += 32) sel[(int)(keys[r] & 0xffffffffu)] = 1;
    __syncwarp();
    int base = 0;
    for (int j0 = 0; j0 < tn; j0 += 32) {
        const int j = j0 + lane;
        const bool f = (j < tn) && sel[j];
        if (mask_row && j < tn) mask_row[j] = f ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) idx_row[base + __popc(bal & ((1u << lane) - 1u))] = j;
        base += __popc(bal);
    }
}

// K1d': 8 query-block rows per CTA (one warp per row for softmax and top-k).
//   phase 1, all threads: s[r][j] = (sum_c qp[r][c] * kp[j][c], c ascending from 0) * inv_sqrt_d
//            (matrix.hpp:111-118 + 272-277), one column j per thread, 8 interleaved row chains;
//   phase 2, warp r:    m = max, e = expf(s - m), sum serially over j ascending (lane 0),
//            inv = 1 / sum, pc = e * inv (matrix.hpp:144-152), then top-kappa.
// Dynamic smem: 8*tn floats + 8*(npow2*8 + tn) bytes + 8*d floats.
constexpr int RROWS = 8;
__host__ __device__ __forceinline__ int rr_ldv(int tn) { return ((tn + 3) & ~3) + 4; }
template <int TK>  // 0: bitonic top-k; otherwise register top-k with TK keys per lane
__global__ void __launch_bounds__(256, 3) router_rows_kernel(const float* __restrict__ qp, const float* __restrict__ kp,
                                                          int kp_t, float inv_sqrt_d, int tm, int tn, int d, int kappa, int npow2,
                                                          float* __restrict__ pc_out, uint8_t* __restrict__ mask_out,
                                                          int32_t* __restrict__ idx_out) {
    extern __shared__ __align__(16) uint8_t smem[];
    // [8][ldv]: rows padded by 4 floats so the 8 rows' float4 at the same column fall in
    // distinct banks (the serial row sums below read them across lanes)
    const int ldv = rr_ldv(tn);
    float* vals = reinterpret_cast<float*>(smem);
    float* sq = vals + RROWS * ldv;                      // [8][d]
    uint8_t* keyb = reinterpret_cast<uint8_t*>(sq + RROWS * d);
    // per-row top-k scratch: 64-bit sort keys for the bitonic path, selection flags otherwise
    const size_t key_stride = TK > 0 ? (((size_t)tn + 15) & ~size_t(15)) + 512 : (((size_t)npow2 * 8 + tn + 15) & ~size_t(15));
    const int i0 = blockIdx.x * RROWS;
    const int64_t bh = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nrows = min(RROWS, tm - i0);
    {  // the CTA's query rows (contiguous): all loads in flight at once
        const int nq = nrows * d;
        stage_copy<8>(sq, qp + (bh * tm + i0) * (int64_t)d, nq, tid, 256);
        for (int e = nq + tid; e < RROWS * d; e += 256) sq[e] = 0.0f;
    }
    __syncthreads();
    const float* kpb = kp + bh * (int64_t)tn * d;  // row-major [tn][d]
    if (kp_t) {
        const int tnp = (tn + 3) & ~3;  // transposed key rows are padded to whole float4s
        const float* kpt = kp + bh * (int64_t)tnp * d;
        // same 4 x 4 register tile over the transposed keys [d][tn]: for each feature c the
        // lanes read 4 consecutive keys each (one coalesced 512-B row per warp); each chain
        // still accumulates over c ascending with separate mul and add
        const int rg = tid >> 7;
        for (int jg = tid & 127; jg * 4 < tn; jg += 128) {
            float acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
            // pointer-stepped (d and tn are run-time: recomputing 64-bit addresses per step
            // cost more instructions than the FP work, ncu source page)
            const float4* kq = reinterpret_cast<const float4*>(kpt + jg * 4);
            const size_t kstep = (size_t)tnp / 4;  // one feature row of keys, in float4
            const float* sqr = sq + rg * 4 * d;
#pragma unroll 2
            for (int c = 0; c < d; c += 4) {
                float4 kv[4], qv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) kv[u] = __ldg(kq + u * kstep);
                kq += 4 * kstep;
#pragma unroll
                for (int a = 0; a < 4; ++a) qv[a] = *reinterpret_cast<const float4*>(sqr + a * d + c);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const float qa[4] = {qv[a].x, qv[a].y, qv[a].z, qv[a].w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        // products as packed FMUL2 (two IEEE-rounded lanes), sums as scalar FADD
                        // (a packed FADD2 fed by an FMUL2 is contracted to FFMA2 by ptxas, even
                        // from explicit .rn PTX: not the reference's two roundings)
                        const float2 q2 = make_float2(qa[u], qa[u]);
                        const float2 p01 = __fmul2_rn(q2, make_float2(kv[u].x, kv[u].y));
                        const float2 p23 = __fmul2_rn(q2, make_float2(kv[u].z, kv[u].w));
                        acc[a][0] = __fadd_rn(acc[a][0], p01.x);
                        acc[a][1] = __fadd_rn(acc[a][1], p01.y);
                        acc[a][2] = __fadd_rn(acc[a][2], p23.x);
                        acc[a][3] = __fadd_rn(acc[a][3], p23.y);
                    }
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (jg * 4 + b < tn) vals[(rg * 4 + a) * ldv + jg * 4 + b] = __fmul_rn(acc[a][b], inv_sqrt_d);
        }
    } else if ((tn & 3) == 0 && (d & 3) == 0) {
        // register tile: 4 rows x 4 columns per thread, 16 independent serial chains; each
        // loaded qp / kp value feeds 4 products (shared-memory traffic 1/4 of the naive loop)
        const int rg = tid >> 7;  // rows rg*4 .. rg*4+3
        for (int jg = tid & 127; jg * 4 < tn; jg += 128) {
            float acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
            const float* k0 = kpb + (int64_t)(jg * 4) * d;
            for (int c = 0; c < d; c += 4) {
                float4 kv[4], qv[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) kv[b] = *reinterpret_cast<const float4*>(k0 + (int64_t)b * d + c);
#pragma unroll
                for (int a = 0; a < 4; ++a) qv[a] = *reinterpret_cast<const float4*>(sq + (rg * 4 + a) * d + c);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        acc[a][b] = __fadd_rn(acc[a][b], __fmul_rn(qv[a].x, kv[b].x));
                        acc[a][b] = __fadd_rn(acc[a][b], __fmul_rn(qv[a].y, kv[b].y));
                        acc[a][b] = __fadd_rn(acc[a][b], __fmul_rn(qv[a].z, kv[b].z));
                        acc[a][b] = __fadd_rn(acc[a][b], __fmul_rn(qv[a].w, kv[b].w));
                    }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) vals[(rg * 4 + a) * ldv + jg * 4 + b] = __fmul_rn(acc[a][b], inv_sqrt_d);
        }
    } else
    for (int j = tid; j < tn; j += 256) {
        float acc[RROWS];
#pragma unroll
        for (int r = 0; r < RROWS; ++r) acc[r] = 0.0f;
        const float* kr = kpb + (int64_t)j * d;
        for (int c0 = 0; c0 < d; c0 += 16) {
            float kv[16];
            if ((d & 15) == 0) {
#pragma unroll
                for (int u = 0; u < 16; u += 4) {
                    const float4 t = *reinterpret_cast<const float4*>(kr + c0 + u);
                    kv[u] = t.x;
                    kv[u + 1] = t.y;
                    kv[u + 2] = t.z;
                    kv[u + 3] = t.w;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) kv[u] = (c0 + u < d) ? kr[c0 + u] : 0.0f;
            }
            const int cn = min(16, d - c0);
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (u < cn) {
#pragma unroll
                    for (int r = 0; r < RROWS; ++r) acc[r] = __fadd_rn(acc[r], __fmul_rn(sq[r * d + c0 + u], kv[u]));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RROWS; ++r) vals[r * ldv + j] = __fmul_rn(acc[r], inv_sqrt_d);
    }
    __syncthreads();
    const int i = i0 + warp;
    float* v = vals + warp * ldv;
    if (warp < nrows) {
        float m = -INFINITY;
        for (int j = lane; j < tn; j += 32) m = fmaxf(m, v[j]);
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        for (int j = lane; j < tn; j += 32) v[j] = expf_glibc(__fsub_rn(v[j], m));
    }
    __syncthreads();
    // serial sums, j ascending (matrix.hpp:148-149): lane r of warp 0 walks row r, so one warp
    // instruction advances all the CTA's rows (the chains' latency is the same as one per warp)
    float* rinv = sq;  // the query rows are no longer needed
    if (warp == 0 && lane < nrows) {
        const float* vr = vals + lane * ldv;
        float sum = 0.0f;
        int j = 0;
        for (; j + 4 <= tn; j += 4) {
            const float4 t = *reinterpret_cast<const float4*>(vr + j);
            sum = __fadd_rn(sum, t.x);
            sum = __fadd_rn(sum, t.y);
            sum = __fadd_rn(sum, t.z);
            sum = __fadd_rn(sum, t.w);
        }
        for (; j < tn; ++j) sum = __fadd_rn(sum, vr[j]);
        rinv[lane] = __fdiv_rn(1.0f, sum);
    }
    __syncthreads();
    if (warp >= nrows) return;
    float inv = rinv[warp];
    for (int j = lane; j < tn; j += 32) {
        const float p = __fmul_rn(v[j], inv);
        v[j] = p;
        if (pc_out) pc_out[(bh * tm + i) * (int64_t)tn + j] = p;
    }
    __syncwarp();
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(keyb + warp * key_stride);
    uint8_t* mrow = mask_out ? mask_out + (bh * tm + i) * (int64_t)tn : nullptr;
    int32_t* irow = idx_out + (bh * tm + i) * (int64_t)kappa;
    if constexpr (TK > 0) {
        uint8_t* selb = reinterpret_cast<uint8_t*>(keys);
        unsigned long long* cand = reinterpret_cast<unsigned long long*>(selb + (((size_t)tn + 15) & ~size_t(15)));
        if (kappa <= 32) warp_topk_cand<1>(v, tn, kappa, mrow, irow, selb, cand);
        else if (kappa <= 64) warp_topk_cand<2>(v, tn, kappa, mrow, irow, selb, cand);
        else warp_topk_small<TK>(v, tn, kappa, mrow, irow, selb);
    }
    else warp_topk_row(v, tn, kappa, keys, npow2, mrow, irow);
}

size_t router_rows_smem(int tn, int d, bool radix) {
    const size_t ldv = (size_t)rr_ldv(tn);
    int npow2 = 1;
    while (npow2 < tn) npow2 <<= 1;
    const size_t key_stride = radix ? (((size_t)tn + 15) & ~size_t(15)) + 512 : (((size_t)npow2 * 8 + tn + 15) & ~size_t(15));
    return (size_t)RROWS * ldv * 4 + (size_t)RROWS * d * 4 + RROWS * key_stride + 16;
}

// hard_topk alone on a caller-given score matrix (sla2_hard_topk).
__global__ void topk_only_kernel(const float* __restrict__ pc, int tm, int tn, int kappa, int npow2,
                                 uint8_t* __restrict__ mask_out, int32_t* __restrict__ idx_out) {
    extern __shared__ __align__(16) uint8_t smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    float* vals = reinterpret_cast<float*>(keys + npow2);
    uint8_t* sel = reinterpret_cast<uint8_t*>(vals + tn);
    __shared__ int warp_cnt[32];
    const int i = blockIdx.x;
    const int64_t bh = blockIdx.y;
    for (int j = threadIdx.x; j < tn; j += blockDim.x) vals[j] = pc[(bh * tm + i) * (int64_t)tn + j];
    __syncthreads();
    topk_row(vals, tn, kappa, keys, npow2, mask_out ? mask_out + (bh * tm + i) * (int64_t)tn : nullptr,
             idx_out + (bh * tm + i) * (int64_t)kappa, sel, warp_cnt);
}

// Mask -> per-row ascending index lists with counts (sla2_sparse_fwd with a caller mask).
// Rows with no kept block set *empty_flag (the reference throws shape_error, attention.hpp:442-447).
__global__ void mask_to_idx_kernel(const uint8_t* __restrict__ mask, int tn, int32_t* __restrict__ idx,
                                   int32_t* __restrict__ cnt, int* __restrict__ empty_flag) {
    const int64_t row = blockIdx.x;
    if (threadIdx.x != 0) return;
    int n = 0;
    for (int j = 0; j < tn; ++j)
        if (mask[row * tn + j]) idx[row * (int64_t)tn + n++] = j;
    cnt[row] = n;
    if (n == 0) atomicExch(empty_flag, 1);
}

// ---------------------------------------------------------------------------------------------
// host launchers
template <typename T>
static void colmean_t(const void* k, const CUtensorMap* tmk, float* mu, int BH, int N, int d, cudaStream_t st,
                      int* launches) {
    constexpr int COLS = 128 / sizeof(T);
    if (sizeof(T) == 2 && tmk && d % cmt::COLS == 0) {
        // (padding the shared memory so no other CTA shares the SM measured no faster)
        const int smem = (cmt::NST + cmt::NTS) * cmt::TILE;
        ensure_smem_attr((const void*)colmean_tr_kernel, (int)(smem));
        colmean_tr_kernel<<<dim3(d / cmt::COLS, BH), 160, smem, st>>>(*tmk, mu, N, d);
    } else if (tmk && N % cm::ROWS == 0 && d % COLS == 0) {
        const int smem = cm::NST * cm::ROWS * 128;
        ensure_smem_attr((const void*)colmean_tma_kernel<T>, (int)(smem));
        colmean_tma_kernel<T><<<dim3(d / COLS, BH), (COLS / 32 + 1) * 32, smem, st>>>(*tmk, mu, N, d);
    } else {
        colmean_exact_kernel<T><<<dim3((d + 31) / 32, BH), 32, 0, st>>>((const T*)k, mu, N, d);
    }
    ++*launches;
}

// Pool then project. With d % 16 == 0 (every shipped config) pooling writes xbar to `scratch`
// and project_kernel reuses P from shared memory across 32 rows; otherwise the per-block
// kernel projects in place.
// Returns true when xp was written transposed ([BH][d][nrows]; only with want_t and the
// split path).
template <typename T>
static bool launch_pool_project(const T* x, const float* mu, const float* proj, float* xp, int N, int d, int H,
                                int block, int BH, float* scratch, cudaStream_t st, int* launches,
                                bool want_t = false, __nv_bfloat16* phi_out = nullptr) {
    const size_t smem = ((d * sizeof(float) + 15) & ~size_t(15)) + (size_t)block * d * sizeof(T);
    if (smem > 48 * 1024) cudaFuncSetAttribute(pool_project_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const bool split = scratch && (d % 16 == 0) && ((size_t)d * d + 32 * d) * 4 <= 200 * 1024;
    // phi(Q) fused only where phiq_kernel would run: bf16, d = 128, whole warps of 16-lane rows
    const bool phi = phi_out && sizeof(T) == 2 && d == 128;
    pool_project_kernel<T><<<dim3((N + block - 1) / block, BH), d, smem, st>>>(x, mu, proj, xp, N, d, H, block,
                                                                  split ? scratch : nullptr, phi ? phi_out : nullptr);
    ++*launches;
    if (split) {
        const int nrows = (N + block - 1) / block;
        launch_project(scratch, proj, xp, nrows, d, H, BH, want_t ? 1 : 0, st);
        ++*launches;
        return want_t;
    }
    return false;
}

template <typename T>
static cudaError_t router_front_t(const RouterLaunch& a, cudaStream_t st, int* launches) {
    const int BH = (int)(a.B * a.H);
    // The exact column mean is a serial chain on a few SMs: run it on a side stream,
    // concurrently with the query-side pooling/projection, and join before the key side.
    // highest priority: the block scheduler must place the colmean CTAs (the critical path)
    // ahead of the query-side pooling grid launched right after them
    cudaStream_t side = aux_stream(2, +1);
    cudaEvent_t ev_fork = aux_event(30), ev_join = aux_event(31);
    bool forked = false;
    if (a.mu_out) {
        if (a.exact_mu) {
            cudaEventRecord(ev_fork, st);
            cudaStreamWaitEvent(side, ev_fork, 0);
            colmean_t<T>(a.k, a.tm_kcol, a.mu_out, BH, a.N, a.d, side, launches);
            cudaEventRecord(ev_join, side);
            timeline_mark(4, side);
            if (a.mu_ready) cudaEventRecord(a.mu_ready, side);
            forked = true;
        } else {
            // tree-reduced mean, also beside the query side
            cudaEventRecord(ev_fork, st);
            cudaStreamWaitEvent(side, ev_fork, 0);
            const int rows_per = 256;
            const int nch = (a.N + rows_per - 1) / rows_per;
            colmean_partial_kernel<T><<<dim3(nch, BH), a.d, 0, side>>>((const T*)a.k, a.mu_part, a.N, a.d, rows_per);
            colmean_finish_kernel<<<BH, a.d, 0, side>>>(a.mu_part, a.mu_out, nch, a.N, a.d);
            *launches += 2;
            cudaEventRecord(ev_join, side);
            timeline_mark(4, side);
            if (a.mu_ready) cudaEventRecord(a.mu_ready, side);
            forked = true;
        }
    }
    // the query pooling also writes phi(Q) (one read of Q) when it can; else phiq_kernel
    const bool phi_fused = a.phiq_out && sizeof(T) == 2 && a.d == 128;
    launch_pool_project<T>((const T*)a.q, nullptr, a.proj_q, a.qp, a.N, a.d, a.H, a.bq, BH, a.qbar, st, launches,
                           false, phi_fused ? (__nv_bfloat16*)a.phiq_out : nullptr);
    if (a.phiq_out && !phi_fused) launch_phiq(a.q, a.phiq_out, (int64_t)BH * a.N, st, launches);
    timeline_mark(5, st);
    if (a.query_done) cudaEventRecord(a.query_done, st);
    if (forked) cudaStreamWaitEvent(st, ev_join, 0);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t router_back_t(const RouterLaunch& a, cudaStream_t st, int* launches) {
    const int BH = (int)(a.B * a.H);
    const int tm = (a.N + a.bq - 1) / a.bq, tn = (a.N + a.bk - 1) / a.bk;
    int npow2 = 1;
    while (npow2 < tn) npow2 <<= 1;
    // register radix top-k for tn <= 2048 (any kappa), bitonic in shared memory beyond
    const int tk = tn <= 32 * 16 ? 16 : (tn <= 32 * 64 ? 64 : 0);
    const size_t rsm = router_rows_smem(tn, a.d, tk > 0);
    const bool tile_ok = rsm <= 220 * 1024 && (a.d & 3) == 0;  // any tn: transposed rows are padded
    bool kp_t;
    if (a.kbar_ready) {
        // pooled keys already in kbar (launch_kprep, d = 128): project only
        launch_project(a.kbar, a.proj_k, a.kp, tn, a.d, a.H, BH, tile_ok ? 1 : 0, st);
        ++*launches;
        kp_t = tile_ok;
    } else {
        kp_t = launch_pool_project<T>((const T*)a.k, a.smooth ? a.mu_out : nullptr, a.proj_k, a.kp, a.N, a.d, a.H,
                                      a.bk, BH, a.kbar, st, launches, tile_ok);
    }
    if (rsm <= 220 * 1024) {
        const dim3 grid((tm + RROWS - 1) / RROWS, BH);
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
            kern<<<grid, 256, rsm, st>>>(a.qp, a.kp, kp_t ? 1 : 0, a.inv_sqrt_d, tm, tn, a.d, a.kappa, npow2,
                                         a.pc_out, a.mask_out, a.idx_out);
        };
        if (tk == 16) go(router_rows_kernel<16>);
        else if (tk == 64) go(router_rows_kernel<64>);
        else go(router_rows_kernel<0>);
    } else {
        const size_t smem = npow2 * 8 + tn * 4 + a.d * 4 + tn + 16;
        cudaFuncSetAttribute(router_scores_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        router_scores_topk_kernel<<<dim3(tm, BH), 256, smem, st>>>(a.qp, a.kp, a.inv_sqrt_d, tm, tn, a.d, a.kappa,
                                                                    npow2, a.pc_out, a.mask_out, a.idx_out);
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_router_front(const RouterLaunch& a, cudaStream_t st, int* launches) {
    return a.bf16 ? router_front_t<__nv_bfloat16>(a, st, launches) : router_front_t<float>(a, st, launches);
}
cudaError_t launch_router_back(const RouterLaunch& a, cudaStream_t st, int* launches) {
    return a.bf16 ? router_back_t<__nv_bfloat16>(a, st, launches) : router_back_t<float>(a, st, launches);
}
cudaError_t launch_router(const RouterLaunch& a, cudaStream_t st, int* launches) {
    const cudaError_t e = launch_router_front(a, st, launches);
    return e != cudaSuccess ? e : launch_router_back(a, st, launches);
}

cudaError_t launch_colmean(const void* k, const CUtensorMap* tmk, bool bf16, float* mu, int BH, int N, int d,
                           cudaStream_t st, int* launches) {
    if (bf16) colmean_t<__nv_bfloat16>(k, tmk, mu, BH, N, d, st, launches);
    else colmean_t<float>(k, tmk, mu, BH, N, d, st, launches);
    return cudaGetLastError();
}

cudaError_t launch_topk_only(const float* pc, int BH, int tm, int tn, int kappa, uint8_t* mask, int32_t* idx,
                             cudaStream_t st, int* launches) {
    int npow2 = 1;
    while (npow2 < tn) npow2 <<= 1;
    const size_t smem = npow2 * 8 + tn * 4 + tn + 16;
    if (smem > 48 * 1024) cudaFuncSetAttribute(topk_only_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    topk_only_kernel<<<dim3(tm, BH), 256, smem, st>>>(pc, tm, tn, kappa, npow2, mask, idx);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_mask_to_idx(const uint8_t* mask, int rows, int tn, int32_t* idx, int32_t* cnt, int* empty_flag,
                               cudaStream_t st, int* launches) {
    mask_to_idx_kernel<<<rows, 32, 0, st>>>(mask, tn, idx, cnt, empty_flag);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
