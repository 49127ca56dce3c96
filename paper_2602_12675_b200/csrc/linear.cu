// linear.cu -- linear-branch precompute of SLA2 on sm_100a.
//
// Replaces attention.hpp:455-475 of sla2_forward_blockwise:
//   K~ = smooth_k(K); phi(K~) = row_softmax(K~) over the d features     (456-457)
//   z_j = colsum phi(K~_j), h_j = phi(K~_j)^T V_j for every key block j   (459-475)
// The per-query-block complement sum over unselected blocks (495-502) is re-expressed as
// "total minus selected": this file produces the totals Ztot = sum_j z_j and
// Htot = phi(K~)^T V over all N keys; the sparse kernel subtracts the selected part. No per-
// block h_j (d x d) is ever stored.
//
// Kernels:
//   phik_kernel      (SIMT)    phi(K~) rows -> bf16 (or fp32) [BH][N][d], z_j per key block
//   htot_umma_kernel (tcgen05) per (bh, chunk of key blocks): TMA phi(K~)/V tiles, M128 N128
//                              K64 MMAs accumulating in TMEM, partial written once
//   htot_simt_kernel (SIMT)    the fp32 path's partials (any d)
//   lin_reduce_kernel          Htot = sum of partials, Ztot = sum_j z_j (fixed order)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

template <typename T>
__device__ __forceinline__ float ld_f32(const T* p);
template <>
__device__ __forceinline__ float ld_f32<float>(const float* p) {
    return *p;
}
template <>
__device__ __forceinline__ float ld_f32<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}

template <typename OutT>
__device__ __forceinline__ float store_round(OutT* p, float v);
template <>
__device__ __forceinline__ float store_round<float>(float* p, float v) {
    *p = v;
    return v;
}
template <>
__device__ __forceinline__ float store_round<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    *p = b;
    return __bfloat162float(b);
}

// One CTA (4 warps) per (key block j, bh). Each warp owns rows w, w+4, ...; a lane owns the
// features lane, lane+32, ... (d <= 128). z_j is summed over the rows as stored (rounded), so
// Ztot - z_sel matches the operands the tensor cores see.
template <typename InT, typename OutT>
__global__ void __launch_bounds__(128) phik_kernel(const InT* __restrict__ k, const float* __restrict__ mu,
                                                   OutT* __restrict__ phik, float* __restrict__ zblk, int N, int d,
                                                   int bk) {
    const int j = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tn = N / bk;
    __shared__ float zpart[4][128];
    float zacc[4] = {0.f, 0.f, 0.f, 0.f};
    float m4[4];
    for (int u = 0; u < 4; ++u) {
        const int f = lane + 32 * u;
        m4[u] = (mu && f < d) ? mu[bh * d + f] : 0.0f;
    }
    for (int t = warp; t < bk; t += 4) {
        const int64_t row = bh * N + (int64_t)j * bk + t;
        float x[4];
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int f = lane + 32 * u;
            x[u] = (f < d) ? ld_f32(k + row * d + f) - m4[u] : -INFINITY;
            mx = fmaxf(mx, x[u]);
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float s = 0.0f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int f = lane + 32 * u;
            x[u] = (f < d) ? expf(x[u] - mx) : 0.0f;
            s += x[u];
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float inv = 1.0f / s;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int f = lane + 32 * u;
            if (f < d) zacc[u] += store_round(phik + row * d + f, x[u] * inv);
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) zpart[warp][lane + 32 * u] = zacc[u];
    __syncthreads();
    for (int f = threadIdx.x; f < d; f += blockDim.x)
        zblk[(bh * tn + j) * d + f] = ((zpart[0][f] + zpart[1][f]) + zpart[2][f]) + zpart[3][f];
}

// phi(Q) = row softmax of Q over the d = 128 features (attention.hpp:456), rounded to bf16 [BH*N][128]:
// the A operand of the sparse kernel's phi(Q) Hc MMA, which TMA-loads it over its Q tile once
// the last Q K^T has read Q. Runs on the query side of the router, off the critical path.
// 16 lanes per row, 8 features (one 16-byte load / store) per lane.
__global__ void __launch_bounds__(256) phiq_kernel(const __nv_bfloat16* __restrict__ q,
                                                   __nv_bfloat16* __restrict__ phiq, int64_t rows) {
    const int64_t row0 = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 4);
    const int sub = threadIdx.x & 15;
    const bool live = row0 < rows;  // the shuffles below need every lane of the warp
    const int64_t row = live ? row0 : rows - 1;
    const uint4 w = *reinterpret_cast<const uint4*>(q + row * 128 + sub * 8);
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
    float x[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
        x[2 * e] = f.x;
        x[2 * e + 1] = f.y;
    }
    float mx = fmaxf(fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3])), fmaxf(fmaxf(x[4], x[5]), fmaxf(x[6], x[7])));
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float s = 0.0f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"((x[e] - mx) * 1.4426950408889634f));
        x[e] = y;
        s += y;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float inv = 1.0f / s;
    uint4 r;
    r.x = pack_bf16(x[0] * inv, x[1] * inv);
    r.y = pack_bf16(x[2] * inv, x[3] * inv);
    r.z = pack_bf16(x[4] * inv, x[5] * inv);
    r.w = pack_bf16(x[6] * inv, x[7] * inv);
    if (live) *reinterpret_cast<uint4*>(phiq + row * 128 + sub * 8) = r;
}

cudaError_t launch_phiq(const void* q, void* phiq, int64_t rows, cudaStream_t st, int* launches) {
    phiq_kernel<<<(unsigned)((rows + 15) / 16), 256, 0, st>>>((const __nv_bfloat16*)q, (__nv_bfloat16*)phiq, rows);
    ++*launches;
    return cudaGetLastError();
}

// phi = row_softmax over the d features in the reference's exact arithmetic (matrix.hpp:138-155):
// max, e_j = expf(x_j - max) (the glibc port), a serial sum in j order, inv = 1 / sum, e_j * inv;
// x = Q (mu null) or K~ = K - mu (fp32 subtraction, quant.hpp:88-96). For SLA2ForwardSaved's
// q_phi / k_phi (attention.hpp:456-457): one warp per row, fp32 out [rows][d], d <= 128.
template <typename InT>
__global__ void __launch_bounds__(256) phi_exact_kernel(const InT* __restrict__ x, const float* __restrict__ mu,
                                                        float* __restrict__ out, int64_t rows, int N, int d) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int64_t bh = row / N;
    float v[4];
    float mx = -INFINITY;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int f = lane + 32 * u;
        float a = -INFINITY;
        if (f < d) {
            a = (float)x[row * d + f];
            if (mu) a = __fsub_rn(a, mu[bh * d + f]);
            mx = fmaxf(mx, a);
        }
        v[u] = a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (lane + 32 * u < d) ? expf_glibc(__fsub_rn(v[u], mx)) : 0.0f;
    float sum = 0.0f;  // serial, j ascending (every lane runs the same chain)
    for (int f = 0; f < d; ++f) sum = __fadd_rn(sum, __shfl_sync(0xffffffffu, v[f >> 5], f & 31));
    const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (lane + 32 * u < d) out[row * d + lane + 32 * u] = __fmul_rn(v[u], inv);
}

cudaError_t launch_phi_exact(const void* x, bool bf16, const float* mu, float* out, int64_t rows, int N, int d,
                             cudaStream_t st, int* launches) {
    const unsigned grid = (unsigned)((rows + 7) / 8);
    if (bf16)
        phi_exact_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, mu, out, rows, N, d);
    else
        phi_exact_kernel<float><<<grid, 256, 0, st>>>((const float*)x, mu, out, rows, N, d);
    ++*launches;
    return cudaGetLastError();
}

// tcgen05 partial Htot for the bf16 path (d = 128, bk = 64): CTA per (chunk, bh) covering
// `per` key blocks; phi(K~)^T V accumulated in 128 TMEM columns; 4 warps read the 128x128
// fp32 partial back (lane = feature f) and store it.
namespace ht {
constexpr int D = 128, BK = 64, NS = 4;
constexpr uint32_t TILE = BK * D * 2;
constexpr uint32_t SMEM = NS * 2 * TILE + 1024;
}  // namespace ht

__global__ void __launch_bounds__(128, 1)
    htot_umma_kernel(const __grid_constant__ CUtensorMap tmPhi, const __grid_constant__ CUtensorMap tmV,
                     float* __restrict__ hpart, int N, int per, int nchunk) {
    using namespace ht;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[NS], empty[NS], done;
    __shared__ uint32_t tbase;
    const int chunk = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tn = N / BK;
    const int j0 = chunk * per;
    const int nblk = min(per, tn - j0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tbase, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    auto sA = [&](int s) { return smem + s * 2 * TILE; };
    auto sB = [&](int s) { return smem + s * 2 * TILE + TILE; };
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmPhi);
        tma_prefetch_desc(&tmV);
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NS;
            if (b >= NS) mbar_wait(&empty[s], ((b / NS) - 1) & 1);
            const int row = (int)(bh * N + (int64_t)(j0 + b) * BK);
            mbar_arrive_expect_tx(&full[s], 2 * TILE);
            tma_load_2d(sA(s), &tmPhi, 0, row, &full[s]);
            tma_load_2d(sA(s) + 8192, &tmPhi, 64, row, &full[s]);
            tma_load_2d(sB(s), &tmV, 0, row, &full[s]);
            tma_load_2d(sB(s) + 8192, &tmV, 64, row, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t ID = idesc_bf16(128, 128, true, true);
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NS;
            mbar_wait(&full[s], (b / NS) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(sA(s)), bb = smem_u32(sB(s));
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                umma_bf16_ss(tmem, sdesc_sw128(a + ks * 2048, 8192, 1024), sdesc_sw128(bb + ks * 2048, 8192, 1024),
                             ID, (b > 0 || ks > 0));
            umma_commit(&empty[s]);
        }
        umma_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
    __syncwarp();
    tc_fence_after();
    const int f = warp * 32 + lane;
    float* dst = hpart + ((bh * nchunk + chunk) * (int64_t)D + f) * D;
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; c += 4)
            *reinterpret_cast<float4*>(dst + c0 + c) =
                make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]), __uint_as_float(r[c + 2]),
                            __uint_as_float(r[c + 3]));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free(tmem, 128);
}

// Fused phi(K~) + partial Htot for the bf16 path (d = 128, bk = 64): CTA per (chunk of `per`
// key blocks, bh). TMA brings K and V tiles; four warps turn the K tile into phi(K~) in place
// (the same instructions as kprep_kernel: fp32 K - mu, redux max, ex2.approx, shuffle sum,
// __fdividef, bf16 round) and store the rows to global for the sparse kernel; the tcgen05 MMA
// then reads phi(K~) straight from shared memory (no global round trip: K + V read once,
// phi(K~) written once). z_j: the four row-group partials summed in fixed order.
// Warps: 0 TMA, 1 TMEM alloc + MMA issue, 2-5 phi(K~) then the partial's TMEM read-back.
namespace kh {
constexpr int D = 128, BK = 64, NS = 2;  // 2 stages: 64 KB per CTA leaves shared memory for
                                         // the router CTAs running beside it (3 measured slower)
constexpr uint32_t TILE = BK * D * 2;            // 16 KB
constexpr uint32_t SMEM = NS * 2 * TILE + 1024;  // [K -> phi(K~)][V] per stage
}  // namespace kh

__global__ void __launch_bounds__(192, 1)
    kphi_htot_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                     const float* __restrict__ mu, __nv_bfloat16* __restrict__ phik, float* __restrict__ zblk,
                     float* __restrict__ hpart, int N, int per, int nchunk, uint8_t* __restrict__ phi8) {
    using namespace kh;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[NS], phi_ready[NS], empty[NS], done;
    __shared__ uint32_t tbase;
    __shared__ __align__(16) float zpart[4][D];
    const int chunk = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tn = (N + BK - 1) / BK;
    const int j0 = chunk * per;
    const int nblk = min(per, tn - j0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&phi_ready[s], 128);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&tbase, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    auto sK = [&](int s) { return smem + s * 2 * TILE; };
    auto sV = [&](int s) { return smem + s * 2 * TILE + TILE; };
    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmV);
            for (int b = 0; b < nblk; ++b) {
                const int s = b % NS;
                if (b >= NS) mbar_wait(&empty[s], ((b / NS) - 1) & 1);
                const int row = (j0 + b) * BK, hz = (int)bh;  // 3-D maps: rows past N read as zeros
                mbar_arrive_expect_tx(&full[s], 2 * TILE);
                tma_load_3d(sK(s), &tmK, 0, row, hz, &full[s]);
                tma_load_3d(sK(s) + 8192, &tmK, 64, row, hz, &full[s]);
                tma_load_3d(sV(s), &tmV, 0, row, hz, &full[s]);
                tma_load_3d(sV(s) + 8192, &tmV, 64, row, hz, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t ID = idesc_bf16(128, 128, true, true);
            for (int b = 0; b < nblk; ++b) {
                const int s = b % NS;
                mbar_wait(&phi_ready[s], (b / NS) & 1);
                tc_fence_after();
                const uint32_t a = smem_u32(sK(s)), bb = smem_u32(sV(s));
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    umma_bf16_ss(tmem, sdesc_sw128(a + ks * 2048, 8192, 1024),
                                 sdesc_sw128(bb + ks * 2048, 8192, 1024), ID, (b > 0 || ks > 0));
                umma_commit(&empty[s]);
            }
            umma_commit(&done);
        }
    } else {
        // phi(K~): warp g = warp - 2 owns rows 16g .. 16g + 15; lane l owns features 4l .. 4l + 3
        const int g = warp - 2;
        float m[4] = {0.f, 0.f, 0.f, 0.f};  // mu == nullptr: phi of the raw K (smooth = 0)
        if (mu) {
            const float4 t = *reinterpret_cast<const float4*>(mu + bh * D + lane * 4);
            m[0] = t.x;
            m[1] = t.y;
            m[2] = t.z;
            m[3] = t.w;
        }
        // SW128 position of the lane's 8 bytes in row r: atom (l / 16), 16-byte chunk (l % 16) / 2
        const uint32_t atom = (uint32_t)(lane >> 4) * 8192u, ch = (uint32_t)((lane & 15) >> 1),
                       half = (uint32_t)(lane & 1) * 8u;
        for (int b = 0; b < nblk; ++b) {
            const int s = b % NS;
            mbar_wait(&full[s], (b / NS) & 1);
            const uint32_t kb = smem_u32(sK(s));
            const int64_t grow0 = bh * N + (int64_t)(j0 + b) * BK;
            const int cnt = min(BK, N - (j0 + b) * BK);  // keys of this block (ragged tail: fewer)
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            constexpr int U = 4;
            for (int r0 = g * 16; r0 < g * 16 + 16; r0 += U) {
                float xs[U][4], mx[U], sum[U];
                uint32_t addr[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = r0 + u;
                    addr[u] = kb + atom + (uint32_t)r * 128u + ((ch ^ (uint32_t)(r & 7)) << 4) + half;
                    uint32_t w0, w1;
                    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(addr[u]));
                    xs[u][0] = __uint_as_float(w0 << 16);
                    xs[u][1] = __uint_as_float(w0 & 0xffff0000u);
                    xs[u][2] = __uint_as_float(w1 << 16);
                    xs[u][3] = __uint_as_float(w1 & 0xffff0000u);
                    mx[u] = -INFINITY;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        xs[u][e] = __fsub_rn(xs[u][e], m[e]);
                        mx[u] = fmaxf(mx[u], xs[u][e]);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mx[u]) : "f"(mx[u]));
                    sum[u] = 0.0f;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float y;
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"((xs[u][e] - mx[u]) * 1.4426950408889634f));
                        xs[u][e] = y;
                        sum[u] += y;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int u = 0; u < U; ++u) sum[u] += __shfl_xor_sync(0xffffffffu, sum[u], o);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float inv = __fdividef(1.0f, sum[u]);
                    uint32_t w0 = pack_bf16(xs[u][0] * inv, xs[u][1] * inv);
                    uint32_t w1 = pack_bf16(xs[u][2] * inv, xs[u][3] * inv);
                    if (r0 + u >= cnt) w0 = w1 = 0u;  // past N: no key, phi = 0 (adds nothing to Htot)
                    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr[u]), "r"(w0), "r"(w1) : "memory");
                    if (r0 + u < cnt) {
                        if (phi8)  // FP8 P/V mode: only the E4M3 448 phi(K~) rows the sparse kernel reads
                            *reinterpret_cast<uint32_t*>(phi8 + (grow0 + r0 + u) * D + lane * 4) =
                                pack_e4m3x2(__uint_as_float(w0 << 16) * 448.0f, __uint_as_float(w0 & 0xffff0000u) * 448.0f) |
                                (pack_e4m3x2(__uint_as_float(w1 << 16) * 448.0f, __uint_as_float(w1 & 0xffff0000u) * 448.0f)
                                 << 16);
                        else
                            *reinterpret_cast<uint2*>(phik + (grow0 + r0 + u) * D + lane * 4) = make_uint2(w0, w1);
                    }
                    z[0] += __uint_as_float(w0 << 16);
                    z[1] += __uint_as_float(w0 & 0xffff0000u);
                    z[2] += __uint_as_float(w1 << 16);
                    z[3] += __uint_as_float(w1 & 0xffff0000u);
                }
            }
            fence_proxy_async_smem();  // phi(K~) written by threads, read by the tensor core
            mbar_arrive(&phi_ready[s]);
            // z_j = ((z_0 + z_1) + z_2) + z_3 over the four row groups
            *reinterpret_cast<float4*>(&zpart[g][lane * 4]) = make_float4(z[0], z[1], z[2], z[3]);
            named_bar_sync(1, 128);
            if (g == 0) {
                float4 zz;
                float* zo = &zz.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int f = lane * 4 + e;
                    zo[e] = ((zpart[0][f] + zpart[1][f]) + zpart[2][f]) + zpart[3][f];
                }
                *reinterpret_cast<float4*>(zblk + (bh * tn + j0 + b) * D + lane * 4) = zz;
            }
            named_bar_sync(1, 128);
        }
        // the chunk's partial phi(K~)^T V: lane = feature f
        mbar_wait(&done, 0);
        __syncwarp();
        tc_fence_after();
        const int q = warp & 3;  // TMEM lane quarter of this warp
        const int f = q * 32 + lane;
        float* dst = hpart + ((bh * nchunk + chunk) * (int64_t)D + f) * D;
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 64) {
            uint32_t r[64];
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 64; c += 4)
                *reinterpret_cast<float4*>(dst + c0 + c) =
                    make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]), __uint_as_float(r[c + 2]),
                                __uint_as_float(r[c + 3]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free(tmem, 128);
}

// SIMT partial Htot for the fp32 path: CTA per (chunk of `rows` tokens, bh); thread owns
// entries e = tid, tid+256, ... of the d x d matrix; tokens staged through smem.
template <typename InT>
__global__ void __launch_bounds__(256) htot_simt_kernel(const float* __restrict__ phik, const InT* __restrict__ v,
                                                        float* __restrict__ hpart, int N, int d, int rows,
                                                        int nchunk) {
    extern __shared__ float sm[];
    float* sphi = sm;          // [32][d]
    float* sv = sm + 32 * d;   // [32][d]
    const int chunk = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int r0 = chunk * rows, r1 = min(N, r0 + rows);
    const int dd = d * d;
    float acc[64];
    const int nper = (dd + 255) / 256;
    for (int u = 0; u < nper && u < 64; ++u) acc[u] = 0.0f;
    for (int t0 = r0; t0 < r1; t0 += 32) {
        const int nt = min(32, r1 - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < nt * d; e += blockDim.x) {
            const int64_t g = (bh * N + t0) * (int64_t)d + e;
            sphi[e] = phik[g];
            sv[e] = ld_f32(v + g);
        }
        __syncthreads();
        for (int u = 0; u < nper && u < 64; ++u) {
            const int e = threadIdx.x + 256 * u;
            if (e < dd) {
                const int f = e / d, c = e % d;
                float a = acc[u];
                for (int t = 0; t < nt; ++t) a = fmaf(sphi[t * d + f], sv[t * d + c], a);
                acc[u] = a;
            }
        }
    }
    for (int u = 0; u < nper && u < 64; ++u) {
        const int e = threadIdx.x + 256 * u;
        if (e < dd) hpart[(bh * nchunk + chunk) * (int64_t)dd + e] = acc[u];
    }
}

// Htot[bh] = sum_chunk hpart[bh][chunk] (chunk ascending); Ztot[bh] = sum_j zblk[bh][j].
// The first CTAs of a head: Htot, four consecutive elements per thread (float4), up to 12
// partials in flight per thread; the last ceil(d / 32): Ztot. blockDim 256, d * d % 4 == 0.
__global__ void __launch_bounds__(256) lin_reduce_kernel(const float* __restrict__ hpart, const float* __restrict__ zblk,
                                  float* __restrict__ htot, __nv_bfloat16* __restrict__ htot16,
                                  float* __restrict__ ztot, int nchunk, int d, int tn) {
    const int64_t bh = blockIdx.y;
    const int dd = d * d;
    if (blockIdx.x + (d + 31) / 32 < gridDim.x) {
        const int e4 = blockIdx.x * blockDim.x + threadIdx.x;  // float4 index
        if (e4 * 4 >= dd) return;
        const float4* src = reinterpret_cast<const float4*>(hpart + bh * nchunk * (int64_t)dd) + e4;
        const int stride4 = dd / 4;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int c0 = 0; c0 < nchunk; c0 += 12) {  // loads batched, summed in chunk order
            float4 t[12];
#pragma unroll
            for (int u = 0; u < 12; ++u)
                if (c0 + u < nchunk) t[u] = src[(int64_t)(c0 + u) * stride4];
#pragma unroll
            for (int u = 0; u < 12; ++u)
                if (c0 + u < nchunk) {
                    s.x += t[u].x;
                    s.y += t[u].y;
                    s.z += t[u].z;
                    s.w += t[u].w;
                }
        }
        reinterpret_cast<float4*>(htot + bh * dd)[e4] = s;
        if (htot16) {
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(htot16 + bh * dd + e4 * 4);
            h2[0] = __floats2bfloat162_rn(s.x, s.y);
            h2[1] = __floats2bfloat162_rn(s.z, s.w);
        }
        return;
    }
    // Ztot[f] = sum_j z_j[f]: the last ceil(d / 32) CTAs of the head, 32 features x 8 parts each;
    // part p sums j = p, p + 8, ... (16 loads in flight per thread), parts combined in order
    __shared__ float zs[256];
    const int zc = blockIdx.x - (gridDim.x - (d + 31) / 32);
    const int f = zc * 32 + (threadIdx.x & 31), part = threadIdx.x >> 5;
    float s = 0.0f;
    if (f < d) {
        for (int j0 = part; j0 < tn; j0 += 16 * 8) {
            float t[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int j = j0 + u * 8;
                t[u] = j < tn ? zblk[(bh * tn + j) * d + f] : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) s += t[u];
        }
    }
    zs[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < 32 && f < d) {
        float t = 0.0f;
        for (int p = 0; p < 8; ++p) t += zs[p * 32 + threadIdx.x];
        ztot[bh * d + f] = t;
    }
}

// Fused key-side prep for d = 128 (one key block per warp, its bk rows in order):
//   kbar[j][c] = float( (sum_r (double)(K[r][c] - mu[c])) / (double)bk )
//       exactly pool_project_kernel's pooled row (matrix.hpp:180-192: r ascending, fp64 sum,
//       fp32 subtraction first) -- the router's key side then only projects it;
//   phi(K~) rows (row softmax over d, attention.hpp:456) -> bf16 / fp32 store, and
//   z_j = column sum of the stored (rounded) rows.
// K is read once for both (phik_kernel + pool_project_kernel read it twice). The exponential
// is ex2.approx: phi(K~) feeds only the linear branch (tolerance 1e-2) and is rounded to bf16;
// each warp stages its key block in shared memory with one bulk copy (the loop is then free of
// DRAM latency), and the row max is one redux.sync.max.f32;
// Htot and the selected-block sums use the same stored values, so "total minus selected" stays
// consistent. Lane l owns features 4l .. 4l+3. grid (ceil(tn/4), BH), block 128.
template <typename T>
struct kp_vec;
template <>
struct kp_vec<__nv_bfloat16> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&x)[4]) {
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        x[0] = __uint_as_float(w.x << 16);
        x[1] = __uint_as_float(w.x & 0xffff0000u);
        x[2] = __uint_as_float(w.y << 16);
        x[3] = __uint_as_float(w.y & 0xffff0000u);
    }
    static __device__ __forceinline__ void store(__nv_bfloat16* p, float (&x)[4]) {
        const __nv_bfloat162 a = __floats2bfloat162_rn(x[0], x[1]), b = __floats2bfloat162_rn(x[2], x[3]);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&a);
        w.y = *reinterpret_cast<const uint32_t*>(&b);
        *reinterpret_cast<uint2*>(p) = w;
        const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
        x[0] = fa.x;
        x[1] = fa.y;
        x[2] = fb.x;
        x[3] = fb.y;
    }
};
template <>
struct kp_vec<float> {
    static __device__ __forceinline__ void load(const float* p, float (&x)[4]) {
        const float4 w = *reinterpret_cast<const float4*>(p);
        x[0] = w.x;
        x[1] = w.y;
        x[2] = w.z;
        x[3] = w.w;
    }
    static __device__ __forceinline__ void store(float* p, float (&x)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
    }
};

__device__ __forceinline__ float warp_max_f32(float x) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
    return r;
}

// POOL / PHI select the halves: the pooled keys are on the router's critical path (mu -> pooled
// keys -> projection -> scores), phi(K~) / z_j only feed the linear branch, so sla2_forward runs
// the pool-only instance on the router's stream and the phi-only one beside the router's back half.
template <typename T, bool POOL, bool PHI>
__global__ void __launch_bounds__(128) kprep_kernel(const T* __restrict__ k, const float* __restrict__ mu,
                                                    T* __restrict__ phik, float* __restrict__ zblk,
                                                    float* __restrict__ kbar, int N, int bk, int tn) {
    constexpr int D = 128;
    extern __shared__ __align__(128) uint8_t kps[];
    __shared__ uint64_t bar[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * 4 + warp;
    const int64_t bh = blockIdx.y;
    const int cnt = min(bk, N - j * bk);  // rows of this key block (ragged tail: fewer)
    const uint32_t blk_bytes = (uint32_t)(cnt > 0 ? cnt : 0) * D * sizeof(T);  // bytes copied
    T* tile = reinterpret_cast<T*>(kps + (size_t)warp * bk * D * sizeof(T));      // full-block slots
    const int64_t row0 = bh * N + (int64_t)j * bk;
    // the warp's whole key block (bk rows, contiguous in global) in one bulk copy
    if (lane == 0) {
        mbar_init(&bar[warp], 1);
        fence_barrier_init();
    }
    __syncwarp();
    if (j >= tn) return;
    if (lane == 0) {
        mbar_arrive_expect_tx(&bar[warp], blk_bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(tile)),
            "l"(k + row0 * D), "r"(blk_bytes), "r"(smem_u32(&bar[warp]))
            : "memory");
    }
    float m[4] = {0.f, 0.f, 0.f, 0.f};
    if (mu) {
        const float4 t = *reinterpret_cast<const float4*>(mu + bh * D + lane * 4);
        m[0] = t.x;
        m[1] = t.y;
        m[2] = t.z;
        m[3] = t.w;
    }
    double pool[4] = {0.0, 0.0, 0.0, 0.0};
    float z[4] = {0.f, 0.f, 0.f, 0.f};
    T* pr = phik + row0 * D + lane * 4;
    mbar_wait(&bar[warp], 0);
    const T* tr = tile + lane * 4;
    constexpr int U = 4;  // rows interleaved (independent reductions)
    for (int r0 = 0; r0 < bk; r0 += U) {
        float xs[U][4], mx[U], sum[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool real = r0 + u < cnt;
            if (real) kp_vec<T>::load(tr + (r0 + u) * D, xs[u]);
            else xs[u][0] = xs[u][1] = xs[u][2] = xs[u][3] = 0.0f;
            mx[u] = -INFINITY;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (mu) xs[u][e] = __fsub_rn(xs[u][e], m[e]);
                if (POOL && real) pool[e] = __dadd_rn(pool[e], (double)xs[u][e]);  // rows in order (exact pooling)
                mx[u] = fmaxf(mx[u], xs[u][e]);
            }
        }
        if (!PHI) continue;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            mx[u] = warp_max_f32(mx[u]);
            sum[u] = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float y;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"((xs[u][e] - mx[u]) * 1.4426950408889634f));
                xs[u][e] = y;
                sum[u] += y;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < U; ++u) sum[u] += __shfl_xor_sync(0xffffffffu, sum[u], o);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float inv = __fdividef(1.0f, sum[u]);
#pragma unroll
            for (int e = 0; e < 4; ++e) xs[u][e] *= inv;
            if (r0 + u >= cnt) continue;  // ragged tail: no key past N
            kp_vec<T>::store(pr + (int64_t)(r0 + u) * D, xs[u]);  // rounds xs to the stored values
#pragma unroll
            for (int e = 0; e < 4; ++e) z[e] += xs[u][e];
        }
    }
    float* kb = kbar + (bh * tn + j) * D + lane * 4;
    float* zb = zblk + (bh * tn + j) * D + lane * 4;
    if (POOL) {
        float kv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) kv[e] = __double2float_rn(__ddiv_rn(pool[e], (double)cnt));
        *reinterpret_cast<float4*>(kb) = make_float4(kv[0], kv[1], kv[2], kv[3]);
    }
    if (PHI) *reinterpret_cast<float4*>(zb) = make_float4(z[0], z[1], z[2], z[3]);
}

template <bool POOL, bool PHI>
static void kprep_go(const LinearLaunch& a, float* kbar, cudaStream_t st) {
    const int tn = (a.N + a.bk - 1) / a.bk;
    const dim3 g((tn + 3) / 4, (unsigned)a.BH);
    const size_t smem = (size_t)4 * a.bk * 128 * (a.bf16 ? 2 : 4);
    if (a.bf16) {
        cudaFuncSetAttribute(kprep_kernel<__nv_bfloat16, POOL, PHI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        kprep_kernel<__nv_bfloat16, POOL, PHI><<<g, 128, smem, st>>>(
            (const __nv_bfloat16*)a.k, a.mu, (__nv_bfloat16*)a.phik, a.zblk, kbar, a.N, a.bk, tn);
    } else {
        cudaFuncSetAttribute(kprep_kernel<float, POOL, PHI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kprep_kernel<float, POOL, PHI><<<g, 128, smem, st>>>((const float*)a.k, a.mu, (float*)a.phik, a.zblk, kbar,
                                                             a.N, a.bk, tn);
    }
}

cudaError_t launch_kprep(const LinearLaunch& a, float* kbar, cudaStream_t st, int* launches) {
    kprep_go<true, true>(a, kbar, st);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_kpool(const LinearLaunch& a, float* kbar, cudaStream_t st, int* launches) {
    kprep_go<true, false>(a, kbar, st);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_kphi(const LinearLaunch& a, cudaStream_t st, int* launches) {
    kprep_go<false, true>(a, nullptr, st);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_linear_prep(const LinearLaunch& a, cudaStream_t st, int* launches) {
    const int tn = (a.N + a.bk - 1) / a.bk;
    dim3 g1(tn, (unsigned)a.BH);
    if (a.bf16 && a.tm_k && !a.phik_ready) {
        // phi(K~), z_j and the Htot partials in one pass over K and V
        ensure_smem_attr((const void*)kphi_htot_kernel, (int)(kh::SMEM));
        const int per = (tn + a.nchunk - 1) / a.nchunk;
        kphi_htot_kernel<<<dim3(a.nchunk, (unsigned)a.BH), 192, kh::SMEM, st>>>(
            *a.tm_k, *a.tm_v, a.mu, (__nv_bfloat16*)a.phik, a.zblk, a.hpart, a.N, per, a.nchunk, a.phi8);
    } else if (a.bf16) {
        if (!a.phik_ready)
            phik_kernel<__nv_bfloat16, __nv_bfloat16><<<g1, 128, 0, st>>>(
                (const __nv_bfloat16*)a.k, a.mu, (__nv_bfloat16*)a.phik, a.zblk, a.N, a.d, a.bk);
        ensure_smem_attr((const void*)htot_umma_kernel, (int)(ht::SMEM));
        const int per = (tn + a.nchunk - 1) / a.nchunk;
        htot_umma_kernel<<<dim3(a.nchunk, (unsigned)a.BH), 128, ht::SMEM, st>>>(*a.tm_phik, *a.tm_v, a.hpart, a.N,
                                                                                 per, a.nchunk);
    } else {
        if (!a.phik_ready)
            phik_kernel<float, float><<<g1, 128, 0, st>>>((const float*)a.k, a.mu, (float*)a.phik, a.zblk, a.N,
                                                          a.d, a.bk);
        const int rows = (a.N + a.nchunk - 1) / a.nchunk;
        const size_t smem = 2 * 32 * a.d * sizeof(float);
        htot_simt_kernel<float><<<dim3(a.nchunk, (unsigned)a.BH), 256, smem, st>>>(
            (const float*)a.phik, (const float*)a.v, a.hpart, a.N, a.d, rows, a.nchunk);
    }
    // Htot CTAs of 256 threads x 4 elements, plus one Ztot CTA per head (blockDim a multiple of d)
    const int hctas = (a.d * a.d / 4 + 255) / 256;
    lin_reduce_kernel<<<dim3(hctas + (a.d + 31) / 32, (unsigned)a.BH), 256, 0, st>>>(
        a.hpart, a.zblk, a.htot, a.bf16 ? (__nv_bfloat16*)a.htot16 : nullptr, a.ztot, a.nchunk, a.d, tn);
    *launches += (a.phik_ready || (a.bf16 && a.tm_k)) ? 2 : 3;
    return cudaGetLastError();
}

}  // namespace sla2dev
