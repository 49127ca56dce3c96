// quant.cu -- INT8 QAT path of the SLA2 forward on sm_100a (BASELINE configs[2]).
//
// Replaces the quantized branches of block_scores_qk / block_product_pv (attention.hpp:372-415)
// with QuantConfig{8, qk_product, pv_product} (quant.hpp:15-19):
//   quantize (quant.hpp:31-50): per tile, absmax over the WHOLE tile (Q_i: bq x d, K~_j: bk x d,
//     V_j: bk x d, P_ij: bq x bk -- SPEC.md:362), scale = absmax / 127 (fp32), inv = 1 / scale,
//     code = clamp(round-half-away(fl(x * inv)), -127, 127); an all-zero tile gets scale FLT_MIN.
//   quantized_product (quant.hpp:62-83): int32 accumulation, then (float)acc * fl(sA * sB).
//   S = fl(fl((float)acc_qk * fl(sQ * sK)) * inv_sqrt_d)    (attention.hpp:381)
// The codes, scales and S are reproduced exactly (same inputs -> same bits); P comes from a fast
// exp2, so P codes and O_s agree within tolerance, not bitwise. The running max is exact (no
// lazy rescale) because the P tile's absmax -- and so every P code -- depends on it; O is kept in
// fp32 registers as o = o * corr + (float)acc_pv * fl(sP * sV) (attention.hpp:512-529).
// The linear branch (phi(K~)^T V, complement, alpha blend) is the bf16 path's.
//
// Kernels: quant_prep_kernel (codes + scales for Q, K~, V; one CTA per 64-row tile) and
// sla2_sparse_i8_kernel (tcgen05 kind::i8 for Q K~^T and P V, kind::f16 for the linear branch).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

__device__ __forceinline__ int8_t quant_code(float x, float inv) {
    float r = roundf(__fmul_rn(x, inv));  // lround((double)fl(x*inv)): ties away from zero
    r = fminf(fmaxf(r, -127.0f), 127.0f);
    return (int8_t)(int)r;
}

// Codes + scale of one [rows x 128] bf16 tile (rows = 64 or 128): block absmax, then codes.
// kind: 0 = Q (block bq), 1 = K~ (block bk, K - mu), 2 = V (block bk). 16-byte loads, the tile
// held in registers between the absmax and the codes (one read of the input).
template <int ROWS>
__device__ __forceinline__ void quant_tile(const __nv_bfloat16* __restrict__ src, const float* __restrict__ m,
                                           int8_t* __restrict__ dst, float* __restrict__ scale_out) {
    constexpr int IT = ROWS * 128 / 8 / 256;  // uint4 per thread
    __shared__ float red[8];
    float x[IT][8];
    float amax = 0.0f;
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        const int v = threadIdx.x + u * 256;  // uint4 index: row v / 16, columns (v % 16) * 8 ..
        const uint4 w = reinterpret_cast<const uint4*>(src)[v];
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[e]));
            x[u][2 * e] = f.x;
            x[u][2 * e + 1] = f.y;
        }
        if (m) {
            const int c0 = (v & 15) * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) x[u][e] = __fsub_rn(x[u][e], m[c0 + e]);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) amax = fmaxf(amax, fabsf(x[u][e]));
    }
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    amax = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) amax = fmaxf(amax, red[w]);
    const float scale = amax == 0.0f ? 1.17549435e-38f : __fdiv_rn(amax, 127.0f);  // all-zero: FLT_MIN
    const float inv = amax == 0.0f ? 0.0f : __fdiv_rn(1.0f, scale);
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            lo |= (uint32_t)(uint8_t)quant_code(x[u][e], inv) << (8 * e);
            hi |= (uint32_t)(uint8_t)quant_code(x[u][4 + e], inv) << (8 * e);
        }
        reinterpret_cast<uint2*>(dst)[threadIdx.x + u * 256] = make_uint2(lo, hi);
    }
    if (threadIdx.x == 0) *scale_out = scale;
}

__global__ void __launch_bounds__(256) quant_prep_kernel(const __nv_bfloat16* __restrict__ q,
                                                         const __nv_bfloat16* __restrict__ k,
                                                         const __nv_bfloat16* __restrict__ v,
                                                         const float* __restrict__ mu, int N, int bq, int bk,
                                                         int which, int8_t* __restrict__ qc, float* __restrict__ qs,
                                                         int8_t* __restrict__ kc, float* __restrict__ ks,
                                                         int8_t* __restrict__ vc, float* __restrict__ vs) {
    constexpr int d = 128;
    // blockIdx.x enumerates the head's tiles of the selected tensors in the order Q, K~, V
    const int64_t bh = blockIdx.y;
    int blk = blockIdx.x, kind = -1;
    for (int kk = 0; kk < 3 && kind < 0; ++kk) {
        if (!(which & (1 << kk))) continue;
        const int n = N / (kk == 0 ? bq : bk);
        if (blk < n)
            kind = kk;
        else
            blk -= n;
    }
    const int rows = kind == 0 ? bq : bk, nblk = N / rows;
    const __nv_bfloat16* src = (kind == 0 ? q : kind == 1 ? k : v) + (bh * N + (int64_t)blk * rows) * d;
    int8_t* dst = (kind == 0 ? qc : kind == 1 ? kc : vc) + (bh * N + (int64_t)blk * rows) * d;
    float* scale_out = (kind == 0 ? qs : kind == 1 ? ks : vs) + bh * nblk + blk;
    const float* m = (kind == 1 && mu) ? mu + bh * d : nullptr;
    if (rows == 128)
        quant_tile<128>(src, m, dst, scale_out);
    else
        quant_tile<64>(src, m, dst, scale_out);
}

cudaError_t launch_quant_prep(const QuantLaunch& a, cudaStream_t st, int* launches) {
    if (a.d != 128 || (a.bq != 64 && a.bq != 128) || (a.bk != 64 && a.bk != 128)) return cudaErrorInvalidValue;
    const int which = a.which ? a.which : 7;
    const int per_head =
        ((which & 1) ? a.N / a.bq : 0) + ((which & 2) ? a.N / a.bk : 0) + ((which & 4) ? a.N / a.bk : 0);
    quant_prep_kernel<<<dim3(per_head, (unsigned)(a.B * a.H)), 256, 0, st>>>(
        (const __nv_bfloat16*)a.q, (const __nv_bfloat16*)a.k, (const __nv_bfloat16*)a.v, a.smooth ? a.mu : nullptr,
        a.N, a.bq, a.bk, which, a.qc, a.qs, a.kc, a.ks, a.vct, a.vs);
    ++*launches;
    return cudaGetLastError();
}

// ============================================================================ sparse i8 kernel
namespace qp {
constexpr int BQ = 128, BK = 64, D = 128;
constexpr int NSK = 4, NSV = 2;
constexpr uint32_t QC_BYTES = BQ * D;          // 16 KB Q codes
constexpr uint32_t Q_BYTES = BQ * D * 2;       // 32 KB Q bf16 (becomes phi(Q))
constexpr uint32_t KC_BYTES = BK * D;          // 8 KB K~ codes
constexpr uint32_t VC_BYTES = BK * D;          // 8 KB V codes
constexpr uint32_t T16_BYTES = BK * D * 2;     // 16 KB bf16 tile (V or phi(K))
constexpr uint32_t VST_BYTES = VC_BYTES + 2 * T16_BYTES;  // V codes, V bf16, phi(K) bf16
constexpr uint32_t P_BYTES = BQ * 128;         // 16 KB: P codes, 64 B used per 128-B row
constexpr uint32_t HT_BYTES = D * D * 2;
constexpr uint32_t OFF_QC = 0;
constexpr uint32_t OFF_Q = OFF_QC + QC_BYTES;
constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
constexpr uint32_t OFF_V = OFF_K + NSK * KC_BYTES;
constexpr uint32_t OFF_P = OFF_V + NSV * VST_BYTES;
constexpr uint32_t OFF_HT = OFF_P + 2 * P_BYTES;
constexpr uint32_t SMEM_BYTES = OFF_HT + HT_BYTES;
constexpr uint32_t SMEM_ALLOC = SMEM_BYTES + 1024;
constexpr uint32_t TM_S = 0;     // 2 x 64 int32
constexpr uint32_t TM_PV = 128;  // 2 x 128 int32
constexpr uint32_t TM_H = 384;   // 128 fp32 Hsel
constexpr uint32_t TM_L = 0;     // 128 fp32 phi(Q) Hc after the loop
}  // namespace qp
static_assert(qp::SMEM_ALLOC + 2048 <= 232448, "QAT kernel shared memory");

struct SparseI8Params {
    const int32_t* kv_idx;
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* rho;
    const float* ztot;
    const float* zblk;
    const float* qs;
    const float* ks;
    const float* vs;
    __nv_bfloat16* out;
    float* o_s;
    float* o_l;
    float* big_l;
    float* h_blocks;
    float* z_blocks;
    float* s_first;
    const float* htot32;
    int N, H, tm, tn;
    float inv_sqrt_d;
};

__device__ __forceinline__ float fexp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(256, 1)
    sla2_sparse_i8_kernel(const __grid_constant__ CUtensorMap tmQc, const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmKc, const __grid_constant__ CUtensorMap tmVc,
                          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmPhi,
                          const __grid_constant__ CUtensorMap tmHt, const SparseI8Params p) {
    using namespace qp;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_q, bar_ht, bar_phiq, bar_k_full[NSK], bar_k_empty[NSK], bar_v_full[NSV],
        bar_v_empty[NSV], bar_s_full[2], bar_p_full[2], bar_pv_done[2], bar_pv_free[2], bar_lin_ready, bar_lin_done;
    __shared__ uint32_t tmem_base_sh;
    __shared__ float sZc[D];
    __shared__ float sDen[BQ];
    __shared__ float sAmax[2][4];

    const int i = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int h = (int)(bh % p.H);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = p.kv_cnt ? p.kv_cnt[bh * p.tm + i] : p.kappa;
    const int32_t* idx = p.kv_idx + (bh * p.tm + i) * (int64_t)p.kstride;
    const bool linear = nb != p.tn;

    if (threadIdx.x == 0) {
        mbar_init(&bar_q, 1);
        mbar_init(&bar_ht, 1);
        mbar_init(&bar_phiq, 32);
        for (int s = 0; s < NSK; ++s) {
            mbar_init(&bar_k_full[s], 1);
            mbar_init(&bar_k_empty[s], 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(&bar_v_full[s], 1);
            mbar_init(&bar_v_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_s_full[b], 1);
            mbar_init(&bar_p_full[b], 128);
            mbar_init(&bar_pv_done[b], 1);
            mbar_init(&bar_pv_free[b], 128);
        }
        mbar_init(&bar_lin_ready, 128);
        mbar_init(&bar_lin_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    uint8_t* sQc = smem + OFF_QC;
    uint8_t* sQ = smem + OFF_Q;
    uint8_t* sHt = smem + OFF_HT;
    auto sKc = [&](int s) { return smem + OFF_K + s * KC_BYTES; };
    auto sVc = [&](int s) { return smem + OFF_V + s * VST_BYTES; };
    auto sV = [&](int s) { return smem + OFF_V + s * VST_BYTES + VC_BYTES; };
    auto sPh = [&](int s) { return smem + OFF_V + s * VST_BYTES + VC_BYTES + T16_BYTES; };
    auto sPc = [&](int b) { return smem + OFF_P + b * P_BYTES; };
    uint8_t* sHc = smem + OFF_V;  // 32 KB epilogue alias of the V stages (free after the loop)

    if (warp == 0) {
        // Q codes + Q bf16, K~ code ring; one box per lane (bulk-tensor copies issued by one
        // thread complete one after another)
        const uint64_t pol = policy_evict_last();
        const int qrow = (int)(bh * p.N + (int64_t)i * BQ);
        if (lane == 0) mbar_arrive_expect_tx(&bar_q, QC_BYTES + Q_BYTES);
        __syncwarp();
        if (lane == 0) tma_load_2d(sQc, &tmQc, 0, qrow, &bar_q);
        if (lane >= 1 && lane < 5) {
            const int u = lane - 1;
            tma_load_2d(sQ + u * 8192, &tmQ, (u >> 1) * 64, qrow + (u & 1) * 64, &bar_q);
        }
        for (int j = 0; j < nb; ++j) {
            const int s = j % NSK;
            if (lane == 0) {
                if (j >= NSK) mbar_wait(&bar_k_empty[s], ((j / NSK) - 1) & 1);
                mbar_arrive_expect_tx(&bar_k_full[s], KC_BYTES);
                const int krow = (int)(bh * p.N + (int64_t)idx[j] * BK);
                tma_load_2d_hint(sKc(s), &tmKc, 0, krow, &bar_k_full[s], pol);
            }
        }
    } else if (warp == 2) {
        // V codes, V bf16, phi(K) ring; Htot -- one box per lane
        const uint64_t pol = policy_evict_last();
        for (int j = 0; j < nb; ++j) {
            const int s = j % NSV;
            if (lane == 0) {
                if (j >= NSV) mbar_wait(&bar_v_empty[s], ((j / NSV) - 1) & 1);
                mbar_arrive_expect_tx(&bar_v_full[s], linear ? VST_BYTES : VC_BYTES);
                if (j == 0 && linear) mbar_arrive_expect_tx(&bar_ht, HT_BYTES);
            }
            __syncwarp();
            const int krow = (int)(bh * p.N + (int64_t)idx[j] * BK);
            if (lane == 0) tma_load_2d_hint(sVc(s), &tmVc, 0, krow, &bar_v_full[s], pol);
            if (linear) {
                if (lane == 1) tma_load_2d_hint(sV(s), &tmV, 0, krow, &bar_v_full[s], pol);
                if (lane == 2) tma_load_2d_hint(sV(s) + 8192, &tmV, 64, krow, &bar_v_full[s], pol);
                if (lane == 3) tma_load_2d_hint(sPh(s), &tmPhi, 0, krow, &bar_v_full[s], pol);
                if (lane == 4) tma_load_2d_hint(sPh(s) + 8192, &tmPhi, 64, krow, &bar_v_full[s], pol);
                if (j == 0 && lane == 5) tma_load_2d_hint(sHt, &tmHt, 0, (int)(bh * D), &bar_ht, pol);
                if (j == 0 && lane == 6) tma_load_2d_hint(sHt + 16384, &tmHt, 64, (int)(bh * D), &bar_ht, pol);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t ID_QK = idesc_s8(128, 64, false, false);
            constexpr uint32_t ID_PV = idesc_s8(128, 128, false, true);
            constexpr uint32_t ID_HS = idesc_bf16(128, 128, true, true);
            constexpr uint32_t ID_LIN = idesc_bf16(128, 128, false, true);
            mbar_wait(&bar_q, 0);
            tc_fence_after();
            const uint32_t aQ = smem_u32(sQc);
            int nq = 0, nh = 0, np = 0;
            while (np < nb) {
                // QK_n into S[n&1]: S[b] is free once the softmax released it (p_full of n-2)
                if (nq < nb && nq <= np + 1 && mbar_try_wait(&bar_k_full[nq % NSK], (nq / NSK) & 1)) {
                    tc_fence_after();
                    const uint32_t bK = smem_u32(sKc(nq % NSK));
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        umma_s8_ss(tmem + TM_S + (nq & 1) * 64, sdesc_sw128(aQ + ks * 32, 16, 1024),
                                   sdesc_sw128(bK + ks * 32, 16, 1024), ID_QK, ks > 0);
                    umma_commit(&bar_s_full[nq & 1]);
                    umma_commit(&bar_k_empty[nq % NSK]);
                    ++nq;
                }
                if (linear && nh < nb && nh <= np + 1 && mbar_try_wait(&bar_v_full[nh % NSV], (nh / NSV) & 1)) {
                    tc_fence_after();
                    const uint32_t aH = smem_u32(sPh(nh % NSV)), bV = smem_u32(sV(nh % NSV));
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        umma_bf16_ss(tmem + TM_H, sdesc_sw128(aH + ks * 2048, 8192, 1024),
                                     sdesc_sw128(bV + ks * 2048, 8192, 1024), ID_HS, (nh > 0 || ks > 0));
                    ++nh;
                }
                // PV_n into PV[n&1] (fresh int32 tile): needs P_n, V_n, and PV[n&1] drained
                if (np < nq && (!linear || np < nh) && mbar_try_wait(&bar_p_full[np & 1], (np >> 1) & 1)) {
                    if (!linear) mbar_wait(&bar_v_full[np % NSV], (np / NSV) & 1);
                    if (np >= 2) mbar_wait(&bar_pv_free[np & 1], ((np - 2) >> 1) & 1);
                    tc_fence_after();
                    const uint32_t aP = smem_u32(sPc(np & 1)), bVc = smem_u32(sVc(np % NSV));
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks)
                        umma_s8_ss(tmem + TM_PV + (np & 1) * 128, sdesc_sw128(aP + ks * 32, 16, 1024),
                                   sdesc_sw128(bVc + ks * 4096, 8192, 1024), ID_PV, ks > 0);
                    umma_commit(&bar_pv_done[np & 1]);
                    umma_commit(&bar_v_empty[np % NSV]);
                    ++np;
                }
            }
            if (linear) {
                mbar_wait(&bar_lin_ready, 0);
                mbar_wait(&bar_phiq, 0);
                tc_fence_after();
                const uint32_t aQ16 = smem_u32(sQ), bH = smem_u32(sHc);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_bf16_ss(tmem + TM_L, sdesc_sw128(aQ16 + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024),
                                 sdesc_sw128(bH + ks * 2048, 16384, 1024), ID_LIN, ks > 0);
                umma_commit(&bar_lin_done);
            }
        }
    } else if (warp == 3) {
        // Zc, then phi(Q) in place over the bf16 Q tile and its denominators (as sparse_bf16.cu)
        if (linear) {
            const float* zb = p.zblk + bh * (int64_t)p.tn * D + lane * 4;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = 0; j < nb; ++j) {
                const float4 z = *reinterpret_cast<const float4*>(zb + (int64_t)idx[j] * D);
                acc.x += z.x;
                acc.y += z.y;
                acc.z += z.z;
                acc.w += z.w;
            }
            const float4 zt = *reinterpret_cast<const float4*>(p.ztot + bh * D + lane * 4);
            sZc[lane * 4 + 0] = zt.x - acc.x;
            sZc[lane * 4 + 1] = zt.y - acc.y;
            sZc[lane * 4 + 2] = zt.z - acc.z;
            sZc[lane * 4 + 3] = zt.w - acc.w;
            __syncwarp();
            if (p.z_blocks)
                *reinterpret_cast<float4*>(p.z_blocks + (bh * p.tm + i) * D + lane * 4) =
                    make_float4(sZc[lane * 4], sZc[lane * 4 + 1], sZc[lane * 4 + 2], sZc[lane * 4 + 3]);
            mbar_wait(&bar_q, 0);
            __syncwarp();
            const uint32_t qb = smem_u32(sQ);
            for (int u = 0; u < 4; ++u) {
                const int r = lane + 32 * u;
                float qv[128];
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {
                    uint32_t w[4];
                    ld_shared_v4(qb + (ch >> 3) * 16384 + sw128_off(r, (ch & 7) * 8), w[0], w[1], w[2], w[3]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
                        qv[ch * 8 + 2 * e] = f2.x;
                        qv[ch * 8 + 2 * e + 1] = f2.y;
                    }
                }
                float qm = -INFINITY;
#pragma unroll
                for (int f = 0; f < 128; ++f) qm = fmaxf(qm, qv[f]);
                float qsum = 0.0f;
#pragma unroll
                for (int f = 0; f < 128; ++f) {
                    qv[f] = fexp2((qv[f] - qm) * 1.4426950408889634f);
                    qsum += qv[f];
                }
                const float qinv = 1.0f / qsum;
                float den = 0.0f;
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int f = ch * 8 + 2 * e;
                        const __nv_bfloat162 pk = __floats2bfloat162_rn(qv[f] * qinv, qv[f + 1] * qinv);
                        const float2 pr = __bfloat1622float2(pk);
                        den += pr.x * sZc[f] + pr.y * sZc[f + 1];
                        w[e] = *reinterpret_cast<const uint32_t*>(&pk);
                    }
                    st_shared_v4(qb + (ch >> 3) * 16384 + sw128_off(r, (ch & 7) * 8), w[0], w[1], w[2], w[3]);
                }
                sDen[r] = den;
            }
            fence_proxy_async_smem();
            mbar_arrive(&bar_phiq);
        }
    } else {
        // ===================== softmax + P quantization + O accumulation (thread = row) =====================
        const int r = threadIdx.x - 128;
        const int sw = warp - 4;  // softmax warp 0..3
        const uint32_t lane_base = (uint32_t)(sw * 32) << 16;
        const float* qs = p.qs + bh * p.tm;
        const float* ks = p.ks + bh * p.tn;
        const float* vs = p.vs + bh * p.tn;
        const float sQ_ = qs[i];
        float o[128];
#pragma unroll
        for (int c = 0; c < 128; ++c) o[c] = 0.0f;
        float m = -INFINITY, l = 0.0f;
        float corr_prev = 0.0f, spv_prev = 0.0f;
        // consume PV_{j} (lagged): o = fl(fl(o * corr_j) + fl((float)acc * spv_j))
        auto consume_pv = [&](int j, float corr, float spv) {
            mbar_wait(&bar_pv_done[j & 1], (j >> 1) & 1);
            __syncwarp();
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t a[32];
                tmem_ld32(tmem + lane_base + TM_PV + (j & 1) * 128 + c0, a);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    o[c0 + c] = __fadd_rn(__fmul_rn(o[c0 + c], corr), __fmul_rn((float)(int)a[c], spv));
            }
            tc_fence_before();
            mbar_arrive(&bar_pv_free[j & 1]);
        };
        // the block's K and V scales are gathered through its index (two dependent global
        // loads): fetched one block ahead so the round trips leave the S -> P chain
        float ks_n = 0.0f, vs_n = 0.0f;
        if (nb > 0) {
            const int kb0 = idx[0];
            ks_n = ks[kb0];
            vs_n = vs[kb0];
        }
        for (int j = 0; j < nb; ++j) {
            const int b = j & 1;
            const float ks_j = ks_n, vs_j = vs_n;
            if (j + 1 < nb) {
                const int kb1 = idx[j + 1];
                ks_n = ks[kb1];
                vs_n = vs[kb1];
            }
            const float sqk = __fmul_rn(sQ_, ks_j);
            mbar_wait(&bar_s_full[b], (j >> 1) & 1);
            __syncwarp();
            tc_fence_after();
            uint32_t sr[64];
            tmem_ld32(tmem + lane_base + TM_S + b * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
            tmem_ld32(tmem + lane_base + TM_S + b * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
            tmem_ld_wait();
            float s[64];
            float mx = -INFINITY;
#pragma unroll
            for (int t = 0; t < 64; ++t) {
                s[t] = __fmul_rn(__fmul_rn((float)(int)sr[t], sqk), p.inv_sqrt_d);  // attention.hpp:381
                mx = fmaxf(mx, s[t]);
            }
            if (p.s_first && j == 0) {  // parity hook: S of the first kept block, as the reference forms it
                float* sd = p.s_first + ((bh * p.tm + i) * BQ + r) * BK;
                for (int t = 0; t < 64; ++t) sd[t] = s[t];
            }
            const float m_new = fmaxf(m, mx);
            const float corr = fexp2((m - m_new) * 1.4426950408889634f);  // 0 on the first block
            const float mnl = m_new * 1.4426950408889634f;
            float rs = 0.0f, pmax = 0.0f;
#pragma unroll
            for (int t = 0; t < 64; ++t) {
                s[t] = fexp2(fmaf(s[t], 1.4426950408889634f, -mnl));  // p, unquantized
                rs += s[t];
                pmax = fmaxf(pmax, s[t]);
            }
            l = __fadd_rn(__fmul_rn(corr, l), rs);  // attention.hpp:519 (w = 1)
            m = m_new;
            // tile absmax of P over all 128 rows (quant.hpp:37-38 on the bq x bk block)
            for (int off = 16; off > 0; off >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, off));
            if (lane == 0) sAmax[b][sw] = pmax;
            named_bar_sync(2, 128);
            const float amax = fmaxf(fmaxf(sAmax[b][0], sAmax[b][1]), fmaxf(sAmax[b][2], sAmax[b][3]));
            float sP, invP;
            if (amax == 0.0f) {
                sP = 1.17549435e-38f;
                invP = 0.0f;
            } else {
                sP = __fdiv_rn(amax, 127.0f);
                invP = __fdiv_rn(1.0f, sP);
            }
            // P codes: row r, 64 int8 in the first 64 B of a 128-B K-major SW128 row
            const uint32_t prow = smem_u32(sPc(b));
            if (j >= 2) mbar_wait(&bar_pv_done[b], ((j - 2) >> 1) & 1);  // PV_{j-2} read this buffer
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int t = ch * 16 + e * 4;
                    const uint32_t c0 = (uint32_t)(uint8_t)quant_code(s[t], invP);
                    const uint32_t c1 = (uint32_t)(uint8_t)quant_code(s[t + 1], invP);
                    const uint32_t c2 = (uint32_t)(uint8_t)quant_code(s[t + 2], invP);
                    const uint32_t c3 = (uint32_t)(uint8_t)quant_code(s[t + 3], invP);
                    w[e] = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
                }
                st_shared_v4(prow + sw128_off_b(r, ch * 16), w[0], w[1], w[2], w[3]);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(&bar_p_full[b]);
            // fold the previous block's PV now that this block's S is out of the way
            if (j >= 1) consume_pv(j - 1, corr_prev, spv_prev);
            corr_prev = corr;
            spv_prev = __fmul_rn(sP, vs_j);
        }
        if (nb > 0) consume_pv(nb - 1, corr_prev, spv_prev);
        __syncwarp();
        tc_fence_after();

        float alpha = 1.0f, den = 1.0f;
        if (linear) {
            const float x = p.rho[(int64_t)h * p.tm + i];
            float a = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x)));
            alpha = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
            // all HS MMAs are complete: the last PV commit came after them
            mbar_wait(&bar_ht, 0);
            __syncwarp();
            const uint32_t hb = smem_u32(sHc), htb = smem_u32(sHt);
            fence_proxy_async_smem();
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t hs[32];
                tmem_ld32(tmem + lane_base + TM_H + c0, hs);
                tmem_ld_wait();
                if (p.h_blocks) {  // SLA2ForwardSaved h_blocks: fp32 Htot - Hsel, row f = r
                    const float* ht = p.htot32 + bh * D * D + r * D + c0;
                    float* hb_out = p.h_blocks + ((bh * p.tm + i) * D + r) * D + c0;
                    for (int c = 0; c < 32; ++c) hb_out[c] = ht[c] - __uint_as_float(hs[c]);
                }
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const int c = c0 + ch * 8;
                    const uint32_t off = (c >> 6) * 16384 + sw128_off(r, c & 63);
                    uint32_t t[4], o4[4];
                    ld_shared_v4(htb + off, t[0], t[1], t[2], t[3]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 tf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t[e]));
                        o4[e] = pack_bf16(tf.x - __uint_as_float(hs[ch * 8 + 2 * e]),
                                          tf.y - __uint_as_float(hs[ch * 8 + 2 * e + 1]));
                    }
                    st_shared_v4(hb + off, o4[0], o4[1], o4[2], o4[3]);
                }
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(&bar_lin_ready);
            mbar_wait(&bar_phiq, 0);
            den = sDen[r];
            mbar_wait(&bar_lin_done, 0);
            __syncwarp();
            tc_fence_after();
        }
        if (!linear && p.h_blocks) {  // full row: empty complement
            float* hb_out = p.h_blocks + ((bh * p.tm + i) * D + r) * D;
            for (int c = 0; c < D; ++c) hb_out[c] = 0.0f;
            if (r < 32) p.z_blocks[(bh * p.tm + i) * D + r * 4 + 0] = 0.0f, p.z_blocks[(bh * p.tm + i) * D + r * 4 + 1] = 0.0f,
                        p.z_blocks[(bh * p.tm + i) * D + r * 4 + 2] = 0.0f, p.z_blocks[(bh * p.tm + i) * D + r * 4 + 3] = 0.0f;
        }
        const float inv_l = __fdiv_rn(1.0f, l);
        const float inv_den = 1.0f / den;
        const float beta = 1.0f - alpha;
        const int64_t grow = bh * p.N + (int64_t)i * BQ + r;
        __nv_bfloat16* orow = p.out + grow * D;
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t ln[32];
            if (linear) {
                tmem_ld32(tmem + lane_base + TM_L + c0, ln);
                tmem_ld_wait();
            }
            float res[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float os = __fmul_rn(o[c0 + c], inv_l);  // attention.hpp:538
                const float ol = linear ? __uint_as_float(ln[c]) * inv_den : 0.0f;
                res[c] = linear ? alpha * os + beta * ol : os;
                if (p.o_s) {
                    p.o_s[grow * D + c0 + c] = os;
                    p.o_l[grow * D + c0 + c] = ol;
                }
            }
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint4 w;
                w.x = pack_bf16(res[ch * 8 + 0], res[ch * 8 + 1]);
                w.y = pack_bf16(res[ch * 8 + 2], res[ch * 8 + 3]);
                w.z = pack_bf16(res[ch * 8 + 4], res[ch * 8 + 5]);
                w.w = pack_bf16(res[ch * 8 + 6], res[ch * 8 + 7]);
                *reinterpret_cast<uint4*>(orow + c0 + ch * 8) = w;
            }
        }
        if (p.big_l) p.big_l[grow] = m + logf(l);
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 2) tmem_free(tmem, 512);
}

cudaError_t launch_sparse_i8(const SparseI8Launch& a, cudaStream_t st, int* launches) {
    SparseI8Params p;
    p.kv_idx = a.s.kv_idx;
    p.kv_cnt = a.s.kv_cnt;
    p.kstride = a.s.kstride;
    p.kappa = a.s.kappa;
    p.rho = a.s.rho;
    p.ztot = a.s.ztot;
    p.zblk = a.s.zblk;
    p.qs = a.qs;
    p.ks = a.ks;
    p.vs = a.vs;
    p.out = (__nv_bfloat16*)a.s.out;
    p.o_s = a.s.o_s;
    p.o_l = a.s.o_l;
    p.big_l = a.s.big_l;
    p.h_blocks = a.s.h_blocks;
    p.z_blocks = a.s.z_blocks;
    p.s_first = a.s.s_first;
    p.htot32 = a.s.htot;
    p.N = a.s.N;
    p.H = (int)a.s.H;
    p.tm = a.s.tm;
    p.tn = a.s.tn;
    p.inv_sqrt_d = a.s.inv_sqrt_d;
    if (a.s.o_s == nullptr && a.s.o_l != nullptr) return cudaErrorInvalidValue;
    ensure_smem_attr((const void*)sla2_sparse_i8_kernel, (int)(qp::SMEM_ALLOC));
    dim3 grid(a.s.tm, (unsigned)(a.s.B * a.s.H));
    sla2_sparse_i8_kernel<<<grid, 256, qp::SMEM_ALLOC, st>>>(*a.tm_qc, *a.s.tm_q, *a.tm_kc, *a.tm_vct, *a.s.tm_v,
                                                              *a.s.tm_phik, *a.s.tm_ht, p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
