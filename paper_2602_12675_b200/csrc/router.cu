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

// K0, TMA-fed: one CTA per (32-column group, bh). Warp 1 streams [256 rows x 32 cols] tiles
// of K into a 6-deep shared-memory ring with TMA; warp 0 runs the 32 serial add chains out
// of shared memory with register double-buffering, so the chain runs at FADD latency instead
// of DRAM latency. Same order and roundings as colmean_exact_kernel.
namespace cm {
constexpr int ROWS = 256, NST = 6;
}
template <typename T>
__global__ void __launch_bounds__(64) colmean_tma_kernel(const __grid_constant__ CUtensorMap tmK, float* __restrict__ mu,
                                                         int N, int d) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);  // [NST][ROWS][32]
    __shared__ uint64_t full[cm::NST], empty[cm::NST];
    const int cg = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunk = N / cm::ROWS;  // N % 256 == 0 is checked by the launcher
    if (threadIdx.x == 0) {
        for (int s = 0; s < cm::NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 32);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 1) {
        if (lane == 0) {
            tma_prefetch_desc(&tmK);
            for (int c = 0; c < nchunk; ++c) {
                const int s = c % cm::NST;
                if (c >= cm::NST) mbar_wait(&empty[s], ((c / cm::NST) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], cm::ROWS * 32 * sizeof(T));
                tma_load_2d(ring + (size_t)s * cm::ROWS * 32, &tmK, cg * 32, (int)(bh * N + (int64_t)c * cm::ROWS),
                            &full[s]);
            }
        }
        return;
    }
    float acc = 0.0f;
    for (int c = 0; c < nchunk; ++c) {
        const int s = c % cm::NST;
        mbar_wait(&full[s], (c / cm::NST) & 1);
        const T* tile = ring + (size_t)s * cm::ROWS * 32 + lane;
        float a[32], b[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) a[u] = to_f32(tile[u * 32]);
#pragma unroll 1
        for (int r0 = 0; r0 < cm::ROWS; r0 += 64) {
#pragma unroll
            for (int u = 0; u < 32; ++u) b[u] = to_f32(tile[(r0 + 32 + u) * 32]);
#pragma unroll
            for (int u = 0; u < 32; ++u) acc = __fadd_rn(acc, a[u]);
            if (r0 + 64 < cm::ROWS) {
#pragma unroll
                for (int u = 0; u < 32; ++u) a[u] = to_f32(tile[(r0 + 64 + u) * 32]);
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) acc = __fadd_rn(acc, b[u]);
        }
        mbar_arrive(&empty[s]);
    }
    const float inv = __fdiv_rn(1.0f, (float)N);
    mu[bh * d + cg * 32 + lane] = __fmul_rn(acc, inv);
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
                                    float* __restrict__ xp, int N, int d, int H, int block) {
    extern __shared__ float sbar[];
    const int c = threadIdx.x;
    const int g = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int h = (int)(bh % H);
    const T* src = x + (bh * N + (int64_t)g * block) * d + c;
    const float m = mu ? mu[bh * d + c] : 0.0f;
    double acc = 0.0;
    int r = 0;
    for (; r + 16 <= block; r += 16) {  // loads batched ahead of the serial double chain
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = to_f32(src[(int64_t)(r + u) * d]);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, (double)(mu ? __fsub_rn(v[u], m) : v[u]));
    }
    for (; r < block; ++r) {
        float v = to_f32(src[(int64_t)r * d]);
        if (mu) v = __fsub_rn(v, m);
        acc = __dadd_rn(acc, (double)v);
    }
    sbar[c] = __double2float_rn(__ddiv_rn(acc, (double)block));
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
    xp[(bh * (N / block) + g) * d + c] = o;
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
__global__ void __launch_bounds__(256) router_rows_kernel(const float* __restrict__ qp, const float* __restrict__ kp,
                                                          float inv_sqrt_d, int tm, int tn, int d, int kappa, int npow2,
                                                          float* __restrict__ pc_out, uint8_t* __restrict__ mask_out,
                                                          int32_t* __restrict__ idx_out) {
    extern __shared__ __align__(16) uint8_t smem[];
    float* vals = reinterpret_cast<float*>(smem);       // [8][tn]
    float* sq = vals + RROWS * tn;                       // [8][d]
    uint8_t* keyb = reinterpret_cast<uint8_t*>(sq + RROWS * d);
    const size_t key_stride = ((size_t)npow2 * 8 + tn + 15) & ~size_t(15);
    const int i0 = blockIdx.x * RROWS;
    const int64_t bh = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nrows = min(RROWS, tm - i0);
    for (int e = tid; e < RROWS * d; e += 256) {
        const int r = e / d;
        sq[e] = (r < nrows) ? qp[(bh * tm + i0 + r) * (int64_t)d + (e % d)] : 0.0f;
    }
    __syncthreads();
    const float* kpb = kp + bh * (int64_t)tn * d;
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
        for (int r = 0; r < RROWS; ++r) vals[r * tn + j] = __fmul_rn(acc[r], inv_sqrt_d);
    }
    __syncthreads();
    if (warp >= nrows) return;
    const int i = i0 + warp;
    float* v = vals + warp * tn;
    float m = -INFINITY;
    for (int j = lane; j < tn; j += 32) m = fmaxf(m, v[j]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int j = lane; j < tn; j += 32) v[j] = expf_glibc(__fsub_rn(v[j], m));
    __syncwarp();
    float inv = 0.0f;
    if (lane == 0) {  // serial sum, j ascending (matrix.hpp:148-149)
        float sum = 0.0f;
        int j = 0;
        for (; j + 8 <= tn; j += 8) {
            float t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = v[j + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) sum = __fadd_rn(sum, t[u]);
        }
        for (; j < tn; ++j) sum = __fadd_rn(sum, v[j]);
        inv = __fdiv_rn(1.0f, sum);
    }
    inv = __shfl_sync(0xffffffffu, inv, 0);
    for (int j = lane; j < tn; j += 32) {
        const float p = __fmul_rn(v[j], inv);
        v[j] = p;
        if (pc_out) pc_out[(bh * tm + i) * (int64_t)tn + j] = p;
    }
    __syncwarp();
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(keyb + warp * key_stride);
    warp_topk_row(v, tn, kappa, keys, npow2, mask_out ? mask_out + (bh * tm + i) * (int64_t)tn : nullptr,
                  idx_out + (bh * tm + i) * (int64_t)kappa);
}

size_t router_rows_smem(int tn, int d) {
    int npow2 = 1;
    while (npow2 < tn) npow2 <<= 1;
    const size_t key_stride = ((size_t)npow2 * 8 + tn + 15) & ~size_t(15);
    return (size_t)RROWS * tn * 4 + (size_t)RROWS * d * 4 + RROWS * key_stride + 16;
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
    if (tmk && N % cm::ROWS == 0 && d % 32 == 0) {
        const int smem = cm::NST * cm::ROWS * 32 * (int)sizeof(T);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(colmean_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            attr = true;
        }
        colmean_tma_kernel<T><<<dim3(d / 32, BH), 64, smem, st>>>(*tmk, mu, N, d);
    } else {
        colmean_exact_kernel<T><<<dim3((d + 31) / 32, BH), 32, 0, st>>>((const T*)k, mu, N, d);
    }
    ++*launches;
}

template <typename T>
static cudaError_t launch_router_t(const RouterLaunch& a, cudaStream_t st, int* launches) {
    const int BH = (int)(a.B * a.H);
    if (a.mu_out) {
        if (a.exact_mu) {
            colmean_t<T>(a.k, a.tm_kcol, a.mu_out, BH, a.N, a.d, st, launches);
        } else {
            const int rows_per = 256;
            const int nch = (a.N + rows_per - 1) / rows_per;
            colmean_partial_kernel<T><<<dim3(nch, BH), a.d, 0, st>>>((const T*)a.k, a.mu_part, a.N, a.d, rows_per);
            colmean_finish_kernel<<<BH, a.d, 0, st>>>(a.mu_part, a.mu_out, nch, a.N, a.d);
            *launches += 2;
        }
    }
    const int tm = a.N / a.bq, tn = a.N / a.bk;
    pool_project_kernel<T><<<dim3(tm, BH), a.d, a.d * sizeof(float), st>>>((const T*)a.q, nullptr, a.proj_q, a.qp,
                                                                            a.N, a.d, a.H, a.bq);
    pool_project_kernel<T><<<dim3(tn, BH), a.d, a.d * sizeof(float), st>>>(
        (const T*)a.k, a.smooth ? a.mu_out : nullptr, a.proj_k, a.kp, a.N, a.d, a.H, a.bk);
    *launches += 2;
    int npow2 = 1;
    while (npow2 < tn) npow2 <<= 1;
    const size_t rsm = router_rows_smem(tn, a.d);
    if (rsm <= 220 * 1024) {
        cudaFuncSetAttribute(router_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
        router_rows_kernel<<<dim3((tm + RROWS - 1) / RROWS, BH), 256, rsm, st>>>(
            a.qp, a.kp, a.inv_sqrt_d, tm, tn, a.d, a.kappa, npow2, a.pc_out, a.mask_out, a.idx_out);
    } else {
        const size_t smem = npow2 * 8 + tn * 4 + a.d * 4 + tn + 16;
        cudaFuncSetAttribute(router_scores_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        router_scores_topk_kernel<<<dim3(tm, BH), 256, smem, st>>>(a.qp, a.kp, a.inv_sqrt_d, tm, tn, a.d, a.kappa,
                                                                    npow2, a.pc_out, a.mask_out, a.idx_out);
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_router(const RouterLaunch& a, cudaStream_t st, int* launches) {
    return a.bf16 ? launch_router_t<__nv_bfloat16>(a, st, launches) : launch_router_t<float>(a, st, launches);
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
