// sparse_v4.cu -- the persistent fused SLA2 sparse + linear + alpha-blend forward (sm_100a, bf16,
// d = 128, bq = 128, bk = 64): the per-query-block loop of sla2_forward_blockwise
// (attention.hpp:484-558) with block_scores_qk / block_product_pv (372-415), one query block per
// CTA at a time, the next one's loop overlapping the previous one's epilogue.
//
// What changed against sparse_v2.cu (profiles/trace_v2_r02.txt: each 16 us query block lost
// ~3 us at its start because its first P V waited for the previous block's O to be read out,
// which waited for the linear-branch MMA, which waited for Hc):
//  * one 64-key block per step with TWO S buffers (P written as bf16 over S's own columns), so
//    Q K^T(j + 1) runs while the softmax works on S(j) -- no separate P buffers;
//  * that frees the TMEM for TWO O accumulators: query block k accumulates into O[k & 1] while
//    the epilogue of block k - 1 finishes O[(k - 1) & 1] (S0 | S1 | O0 | O1 | Hsel = 512 columns);
//  * the linear term lands in the finished block's O (as v2): with c_r = (1 - a) l_r / (a den_r),
//    out = a / l (O + (c phi(Q)) Hc); A = c phi(Q) is written by the epilogue over the block's own
//    Q buffer (free after its last Q K^T), B = Hc in a slot of the V ring;
//  * Hsel = sum_sel phi(K~_j)^T V_j (single buffer) is issued as soon as the epilogue of the
//    previous block has read its Hsel, so the next block's Q K^T / P V never wait for it.
//
// Warp roles (384 threads, one CTA per SM):
//   warp 0      TMA: Q (two buffers), K ring (one 64-key block per slot), one box per lane
//   warp 1      MMA issuer
//   warp 2      TMEM allocator; TMA: V / phi(K~) ring (+ one Hc slot per query block)
//   warp 3      Zc = Ztot - sum_sel z_j per query block
//   warps 4-7   softmax (thread = query row), 64 key columns per step
//   warps 8-11  epilogue of the previous query block (thread = row)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

namespace v4 {
constexpr int BQ = 128, BK = 64, D = 128;
#ifndef SLA2_V4_NK
#define SLA2_V4_NK 3
#define SLA2_V4_NV 3
#endif
constexpr int NK = SLA2_V4_NK, NV = SLA2_V4_NV;
constexpr uint32_t Q_BYTES = BQ * D * 2;     // 32 KB
constexpr uint32_t TILE_BYTES = BK * D * 2;  // 16 KB
constexpr uint32_t VS_BYTES = 2 * TILE_BYTES;  // V + phi(K~), or Hc
constexpr uint32_t OFF_Q = 0, OFF_K = 2 * Q_BYTES, OFF_V = OFF_K + NK * TILE_BYTES;
constexpr uint32_t SMEM = OFF_V + NV * VS_BYTES + 1024;  // 209 KB (+ alignment slack; 2.3 KB static)
constexpr uint32_t TM_S = 0, TM_O = 128, TM_H = 384;     // S(b) at 64 b, O(b) at 128 + 128 b
constexpr float RESCALE_LOG2 = 8.0f;
constexpr int NTHREADS = 384;
}  // namespace v4

struct SparseV4Params {
    const int32_t* kv_idx;
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* rho;
    const float* ztot;
    const float* zblk;
    const __nv_bfloat16* htot16;  // [BH][D][D] bf16 (prefetched per row by the epilogue)
    const __nv_bfloat16* phiq;  // [BH][N][D]
    __nv_bfloat16* out;
    int N, H, tm, tn, ntiles;
    int last_valid;
    float scale_log2;
#ifdef SLA2_TRACE
    unsigned long long* trace;  // [grid][4 query blocks][16 steps][8 events] %globaltimer (analysis build)
#endif
};
#ifdef SLA2_TRACE
__device__ __forceinline__ unsigned long long v4_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define V4_TR(k, j, e) \
    if ((k) < 4 && (j) < 16) p.trace[(((size_t)blockIdx.x * 4 + (k)) * 16 + (j)) * 8 + (e)] = v4_gtimer()
#else
#define V4_TR(k, j, e)
#endif

#ifdef SLA2_FA_WATCHDOG
__device__ __forceinline__ void v4_wait_wd(uint64_t* bar, uint32_t parity, int site) {
    for (long long it = 0; !mbar_try_wait(bar, parity); ++it) {
        if (it == (1ll << 25)) {
            printf("sla2 sparse_v4 HANG block %d warp %d lane %d line %d parity %u\n", blockIdx.x, threadIdx.x >> 5,
                   threadIdx.x & 31, site, parity);
            __trap();
        }
    }
}
#define V4_WAIT(bar, par) v4_wait_wd(bar, par, __LINE__)
#else
#define V4_WAIT(bar, par) mbar_wait(bar, par)
#endif

__device__ __forceinline__ float v4_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <uint32_t N>
__device__ __forceinline__ void v4_reg_alloc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void v4_reg_dealloc() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

struct V4Tile {
    int bh, i, nb;
    bool linear;
    const int32_t* idx;
};
__device__ __forceinline__ V4Tile v4_tile(const SparseV4Params& p, int t) {
    V4Tile r;
    r.bh = t / p.tm;
    r.i = t - r.bh * p.tm;
    r.nb = p.kv_cnt ? p.kv_cnt[t] : p.kappa;
    r.idx = p.kv_idx + (int64_t)t * p.kstride;
    r.linear = r.nb != p.tn;
    return r;
}

__global__ void __launch_bounds__(384, 1)
    sla2_sparse_v4_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmPhi,
                          const SparseV4Params p) {
    using namespace v4;
    extern __shared__ uint8_t v4_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(v4_smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_q_full[2], bar_q_free[2], bar_k_full[NK], bar_k_empty[NK], bar_v_full[NV],
        bar_v_empty[NV], bar_s_full[2], bar_p_full[2], bar_pv_done, bar_tile_done, bar_h_free, bar_lin_ready,
        bar_lin_done, bar_o_free[2], bar_l_full[2], bar_l_free[2], bar_zc_ready[2], bar_zc_free[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(16) float sZc[2][D];
    __shared__ float sL[2][BQ];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = p.ntiles, G = gridDim.x;
    const uint32_t sbase = smem_u32(smem);

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_q_full[b], 1);
            mbar_init(&bar_q_free[b], 1);
            mbar_init(&bar_s_full[b], 1);
            mbar_init(&bar_p_full[b], 4);
            mbar_init(&bar_o_free[b], 4);
            mbar_init(&bar_l_full[b], 4);
            mbar_init(&bar_l_free[b], 4);
            mbar_init(&bar_zc_ready[b], 1);
            mbar_init(&bar_zc_free[b], 4);
        }
        for (int s = 0; s < NK; ++s) {
            mbar_init(&bar_k_full[s], 1);
            mbar_init(&bar_k_empty[s], 1);
        }
        for (int s = 0; s < NV; ++s) {
            mbar_init(&bar_v_full[s], 1);
            mbar_init(&bar_v_empty[s], 1);
        }
        mbar_init(&bar_pv_done, 1);
        mbar_init(&bar_tile_done, 1);
        mbar_init(&bar_h_free, 4);
        mbar_init(&bar_lin_ready, 4);
        mbar_init(&bar_lin_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    // registers: 4 x 56 (TMA / MMA / Zc) + 4 x 152 (softmax) + 4 x 256 (epilogue) <= 12 x 168
    if (warp < 4) {
        v4_reg_dealloc<56>();
        if (warp == 0) {
            // ============ TMA: Q of query block k into buffer k & 1 (free after lin(k - 2)), K ring ============
            if (lane == 0) {
                tma_prefetch_desc(&tmQ);
                tma_prefetch_desc(&tmK);
            }
            const uint64_t pol = policy_evict_last();
            int g = 0, k = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V4Tile T = v4_tile(p, t);
                uint8_t* dq = smem + OFF_Q + (k & 1) * Q_BYTES;
                if (lane == 0) {
                    if (k >= 2) V4_WAIT(&bar_q_free[k & 1], (uint32_t)(((k >> 1) - 1) & 1));
                    mbar_arrive_expect_tx(&bar_q_full[k & 1], Q_BYTES);
                }
                __syncwarp();
                if (lane < 4)
                    tma_load_3d(dq + lane * 8192, &tmQ, (lane >> 1) * 64, T.i * BQ + (lane & 1) * 64, T.bh,
                                &bar_q_full[k & 1]);
                for (int j = 0; j < T.nb; ++j, ++g) {
                    const int s = g % NK;
                    if (lane == 0) {
                        if (g >= NK) V4_WAIT(&bar_k_empty[s], (uint32_t)(((g / NK) - 1) & 1));
                        mbar_arrive_expect_tx(&bar_k_full[s], TILE_BYTES);
                    }
                    __syncwarp();
                    if (lane < 2)
                        tma_load_3d_hint(smem + OFF_K + s * TILE_BYTES + lane * 8192, &tmK, lane * 64, T.idx[j] * BK,
                                         T.bh, &bar_k_full[s], pol);
                }
            }
        } else if (warp == 2) {
            // ============ TMA: V / phi(K~) ring; one slot per query block for the epilogue's Hc ============
            if (lane == 0) {
                tma_prefetch_desc(&tmV);
                tma_prefetch_desc(&tmPhi);
            }
            const uint64_t pol = policy_evict_last();
            int gv = 0;
            for (int t = blockIdx.x; t < nt; t += G) {
                const V4Tile T = v4_tile(p, t);
                for (int j = 0; j <= T.nb; ++j, ++gv) {
                    const int s = gv % NV;
                    if (lane == 0) {
                        if (gv >= NV) V4_WAIT(&bar_v_empty[s], (uint32_t)(((gv / NV) - 1) & 1));
                        if (j == T.nb)
                            mbar_arrive(&bar_v_full[s]);  // the Hc slot: allocated, not loaded
                        else
                            mbar_arrive_expect_tx(&bar_v_full[s], T.linear ? VS_BYTES : TILE_BYTES);
                    }
                    __syncwarp();
                    if (j < T.nb && lane < (T.linear ? 4 : 2))  // lanes 0-1: V halves, 2-3: phi(K~) halves
                        tma_load_3d_hint(smem + OFF_V + s * VS_BYTES + lane * 8192, lane < 2 ? &tmV : &tmPhi,
                                         (lane & 1) * 64, T.idx[j] * BK, T.bh, &bar_v_full[s], pol);
                }
            }
        } else if (warp == 1) {
            // ============ MMA issuer ============
            constexpr uint32_t ID_QK = idesc_bf16(128, 64, false, false);
            constexpr uint32_t ID_PV = idesc_bf16(128, 128, false, true);
            constexpr uint32_t ID_HS = idesc_bf16(128, 128, true, true);
            constexpr uint32_t ID_LIN = idesc_bf16(128, 128, false, true);
            const uint32_t tm = warp_uniform(tmem);
            const uint32_t sb = warp_uniform(sbase);
            const uint64_t dK0 = sdesc_sw128(sb + OFF_K, 16, 1024);
            const uint64_t dV0 = sdesc_sw128(sb + OFF_V, 8192, 1024);
            int gk = 0, gp = 0, gv = 0, k = 0;
            int lin_hc = -1;           // pending lin MMA: V-ring slot of Hc (-1: none)
            bool lin_linear = false;
            auto issue_qk = [&](int kk, int g) {  // S(g & 1) = Q(kk) K^T
                const int s = gk % NK;
                V4_WAIT(&bar_k_full[s], (uint32_t)((gk / NK) & 1));
                tc_fence_after();
                const uint64_t dQ = sdesc_sw128(sb + OFF_Q + (kk & 1) * Q_BYTES, 16, 1024);
                const uint64_t dK = dK0 + (uint64_t)((s * TILE_BYTES) >> 4);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_bf16_ss_w(tm + TM_S + (uint32_t)(g & 1) * 64, dQ + (((ks >> 2) * 16384 + (ks & 3) * 32) >> 4),
                                   dK + (((ks >> 2) * 8192 + (ks & 3) * 32) >> 4), ID_QK, ks > 0);
                umma_commit_w(&bar_s_full[g & 1]);
                umma_commit_w(&bar_k_empty[s]);
                ++gk;
            };
            auto issue_lin = [&](int kk) {  // O(kk & 1) += (c phi(Q)) Hc, then Q(kk & 1) and the Hc slot are free
                V4_WAIT(&bar_lin_ready, (uint32_t)(kk & 1));
                tc_fence_after();
                if (lin_linear) {
                    const uint64_t dA = sdesc_sw128(sb + OFF_Q + (kk & 1) * Q_BYTES, 16, 1024);
                    const uint64_t dB = sdesc_sw128(sb + OFF_V + lin_hc * VS_BYTES, 16384, 1024);
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)
                        umma_bf16_ss_w(tm + TM_O + (uint32_t)(kk & 1) * 128,
                                       dA + (((ks >> 2) * 16384 + (ks & 3) * 32) >> 4), dB + ((ks * 2048) >> 4), ID_LIN, 1);
                }
                umma_commit_w(&bar_lin_done);
                umma_commit_w(&bar_q_free[kk & 1]);
                umma_commit_w(&bar_v_empty[lin_hc]);
                lin_hc = -1;
            };
            int hs_issued = 0, hs_slot[NV];  // Hsel MMAs waiting for the previous block's Hsel read-out
            int hs_n = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V4Tile T = v4_tile(p, t);
                const int nbu = (int)warp_uniform((uint32_t)T.nb);
                const bool lin = T.linear;
                const uint32_t tO = tm + TM_O + (uint32_t)(k & 1) * 128;
                V4_WAIT(&bar_q_full[k & 1], (uint32_t)((k >> 1) & 1));
                tc_fence_after();
                const int g0 = gp;
                issue_qk(k, g0);
                if (nbu > 1) issue_qk(k, g0 + 1);
                bool h_ok = k == 0;  // Hsel(k - 1) read by the epilogue
                hs_issued = 0;
                hs_n = 0;
                auto flush_hsel = [&]() {
#pragma unroll 1
                    for (int u = 0; u < hs_n; ++u) {
                        const uint64_t dV = dV0 + (uint64_t)((hs_slot[u] * VS_BYTES) >> 4);
                        const uint64_t dP = dV + (TILE_BYTES >> 4);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            umma_bf16_ss_w(tm + TM_H, dP + ((ks * 2048) >> 4), dV + ((ks * 2048) >> 4), ID_HS,
                                           (hs_issued > 0 || ks > 0));
                        ++hs_issued;
                        umma_commit_w(&bar_v_empty[hs_slot[u]]);
                    }
                    hs_n = 0;
                };
                for (int j = 0; j < nbu; ++j) {
                    const int g = g0 + j;
                    V4_WAIT(&bar_p_full[g & 1], (uint32_t)((g >> 1) & 1));
                    tc_fence_after();
                    if (j == 0 && k >= 2) {
                        V4_WAIT(&bar_o_free[k & 1], (uint32_t)(((k >> 1) - 1) & 1));  // O(k & 1) read out
                        tc_fence_after();
                    }
                    const int sv = gv % NV;
                    // the slot may be held by the previous block's Hc (freed by its lin MMA) or by a
                    // pending Hsel (freed once the epilogue has read Hsel): keep both moving while waiting
                    while (!mbar_try_wait(&bar_v_full[sv], (uint32_t)((gv / NV) & 1))) {
                        if (lin_hc >= 0 && mbar_test_wait(&bar_lin_ready, (uint32_t)((k - 1) & 1))) issue_lin(k - 1);
                        if (hs_n > 0 && (h_ok || mbar_test_wait(&bar_h_free, (uint32_t)((k - 1) & 1)))) {
                            h_ok = true;
                            tc_fence_after();
                            flush_hsel();
                        }
                    }
                    tc_fence_after();
                    const uint64_t dV = dV0 + (uint64_t)((sv * VS_BYTES) >> 4);
                    const uint32_t tP = tm + TM_S + (uint32_t)(g & 1) * 64;
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        umma_bf16_ts_w(tO, tP + ks * 8, dV + ((ks * 2048) >> 4), ID_PV, (j > 0 || ks > 0));
                    umma_commit_w(&bar_pv_done);
                    if (lane == 0) V4_TR(k, j, 0);
                    ++gp;
                    ++gv;
                    if (j + 2 < nbu) issue_qk(k, g + 2);  // over S(g & 1), after P V(g) read it (in order)
                    if (lane == 0) V4_TR(k, j, 3);
                    if (lin) {
                        hs_slot[hs_n++] = sv;
                        if (!h_ok) h_ok = mbar_test_wait(&bar_h_free, (uint32_t)((k - 1) & 1));
                        if (h_ok || hs_n == NV) {  // the ring cannot hold more pending slots: wait
                            if (!h_ok) {
                                V4_WAIT(&bar_h_free, (uint32_t)((k - 1) & 1));
                                h_ok = true;
                            }
                            tc_fence_after();
                            flush_hsel();
                        }
                    } else {
                        umma_commit_w(&bar_v_empty[sv]);
                    }
                    if (lin_hc >= 0 && mbar_test_wait(&bar_lin_ready, (uint32_t)((k - 1) & 1))) issue_lin(k - 1);
                }
                if (lin && hs_n > 0) {
                    if (!h_ok) V4_WAIT(&bar_h_free, (uint32_t)((k - 1) & 1));
                    tc_fence_after();
                    flush_hsel();
                }
                umma_commit_w(&bar_tile_done);
                if (lane == 0) V4_TR(k, 15, 4);
                if (lin_hc >= 0) issue_lin(k - 1);
                if (lane == 0) V4_TR(k, 15, 5);
                lin_hc = gv % NV;  // this block's Hc slot (allocated by the V producer after its blocks;
                lin_linear = lin;  // the epilogue waits for it before writing Hc)
                ++gv;
            }
            if (lin_hc >= 0) issue_lin(k - 1);
        } else {
            // ============ Zc = Ztot - sum_sel z_j per query block (the linear denominators) ============
            int k = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V4Tile T = v4_tile(p, t);
                const int b = k & 1;
                if (k >= 2) V4_WAIT(&bar_zc_free[b], (uint32_t)(((k >> 1) - 1) & 1));
                if (T.linear) {
                    const float* zb = p.zblk + (int64_t)T.bh * p.tn * D + lane * 4;
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int j0 = 0; j0 < T.nb; j0 += 8) {
                        float4 z[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            z[u] = j0 + u < T.nb ? *reinterpret_cast<const float4*>(zb + (int64_t)T.idx[j0 + u] * D)
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            acc.x += z[u].x;
                            acc.y += z[u].y;
                            acc.z += z[u].z;
                            acc.w += z[u].w;
                        }
                    }
                    const float4 zt = *reinterpret_cast<const float4*>(p.ztot + (int64_t)T.bh * D + lane * 4);
                    *reinterpret_cast<float4*>(&sZc[b][lane * 4]) =
                        make_float4(zt.x - acc.x, zt.y - acc.y, zt.z - acc.z, zt.w - acc.w);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_zc_ready[b]);
            }
        }
    } else if (warp < 8) {
        v4_reg_dealloc<152>();
        // ============ softmax: thread = query row r, one key block per step ============
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = p.scale_log2;
        const float2 sc2 = make_float2(sc, sc);
        int g = 0, k = 0;
        for (int t = blockIdx.x; t < nt; t += G, ++k) {
            const V4Tile T = v4_tile(p, t);
            const int nb = T.nb;
            const uint32_t tO = tmem + lane_base + TM_O + (uint32_t)(k & 1) * 128;
            const int jtail = (p.last_valid < BK && T.idx[nb - 1] == p.tn - 1) ? nb - 1 : -1;
            float m = -INFINITY, l = 0.0f;
            for (int j = 0; j < nb; ++j, ++g) {
                V4_WAIT(&bar_s_full[g & 1], (uint32_t)((g >> 1) & 1));
                __syncwarp();
                tc_fence_after();
                if (r == 0) V4_TR(k, j, 1);
                const uint32_t tS = tmem + lane_base + TM_S + (uint32_t)(g & 1) * 64;
                uint32_t sr[64];
                tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                tmem_ld_wait();
                if (j == jtail) {  // ragged N: keys past N in the partial last block
#pragma unroll
                    for (int c = 0; c < 64; ++c)
                        if (c >= p.last_valid) sr[c] = __float_as_uint(-INFINITY);
                }
                float m4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) m4[u] = fmaxf(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
#pragma unroll
                for (int c = 8; c < 64; c += 8) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        m4[u] = fmaxf(m4[u], fmaxf(__uint_as_float(sr[c + 2 * u]), __uint_as_float(sr[c + 2 * u + 1])));
                }
                const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sc;
                if (j == 0) {
                    m = mx;
                } else if (__any_sync(0xffffffffu, mx > m + RESCALE_LOG2)) {
                    // lazy rescale: O must hold P V(g - 1) first
                    const float mnew = fmaxf(m, mx);
                    const float corr = v4_exp2(m - mnew);
                    V4_WAIT(&bar_pv_done, (uint32_t)((g - 1) & 1));
                    __syncwarp();
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 128; c0 += 16) {
                        uint32_t o[16];
                        tmem_ld16(tO + c0, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st16(tO + c0, o);
                    }
                    l *= corr;
                    m = mnew;
                }
                const float2 nm2 = make_float2(-m, -m);
                float2 rs = make_float2(0.f, 0.f);
                uint32_t w[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float2 v2 = __ffma2_rn(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])),
                                                 sc2, nm2);
                    const float2 pe = make_float2(v4_exp2(v2.x), v4_exp2(v2.y));
                    rs = __fadd2_rn(rs, pe);
                    w[e] = pack_bf16(pe.x, pe.y);
                }
                tmem_st32(tS, w);
                l += rs.x + rs.y;
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_p_full[g & 1]);
                if (r == 0) V4_TR(k, j, 2);
            }
            if (k >= 2) V4_WAIT(&bar_l_free[k & 1], (uint32_t)(((k >> 1) - 1) & 1));
            sL[k & 1][r] = l;
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_l_full[k & 1]);
        }
    } else {
        v4_reg_alloc<256>();
        // ============ epilogue of query block k, one block behind the softmax (thread = row r) ============
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int k = 0, gv = 0;  // gv: V-ring position of this block's first kept block
        for (int t = blockIdx.x; t < nt; t += G, ++k) {
            const V4Tile T = v4_tile(p, t);
            const int b = k & 1;
            const int gv_hc = gv + T.nb;  // this block's Hc slot
            gv = gv_hc + 1;
            const bool live = T.i * BQ + r < p.N;
            const int64_t grow = (int64_t)T.bh * p.N + (int64_t)T.i * BQ + r;
            float alpha = 1.0f, cfac = 0.0f;
            uint32_t cq[64];  // phi(Q)_r as packed bf16 pairs, then c phi(Q)_r
            uint4 htr[16];    // Htot row f = r (bf16), loaded before the block's MMAs are done
            if (T.linear) {
                const uint4* ht = reinterpret_cast<const uint4*>(p.htot16 + ((int64_t)T.bh * D + r) * D);
#pragma unroll
                for (int u = 0; u < 16; ++u) htr[u] = ht[u];
                const uint4* pq = reinterpret_cast<const uint4*>(p.phiq + grow * D);
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const uint4 w = live ? pq[u] : make_uint4(0u, 0u, 0u, 0u);
                    cq[4 * u] = w.x;
                    cq[4 * u + 1] = w.y;
                    cq[4 * u + 2] = w.z;
                    cq[4 * u + 3] = w.w;
                }
                const float x = p.rho[(int64_t)(T.bh % p.H) * p.tm + T.i];
                const float a = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x)));
                alpha = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);  // attention.hpp:17-22
            }
            V4_WAIT(&bar_zc_ready[b], (uint32_t)((k >> 1) & 1));
            float den = 1.0f;
            if (T.linear) {  // den = phi(Q)_r . Zc over the bf16 phi(Q) the MMA uses
                float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int e = 0; e < 64; ++e) {
                    const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cq[e]));
                    d2 = __ffma2_rn(f2, *reinterpret_cast<const float2*>(&sZc[b][2 * e]), d2);
                }
                den = d2.x + d2.y;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_zc_free[b]);
            V4_WAIT(&bar_l_full[b], (uint32_t)((k >> 1) & 1));
            const float l = sL[b][r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_l_free[b]);
            if (T.linear) {
                cfac = (live && den > 0.0f) ? (1.0f - alpha) * l / (alpha * den) : 0.0f;
#pragma unroll
                for (int e = 0; e < 64; ++e) {
                    const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cq[e]));
                    cq[e] = pack_bf16(f2.x * cfac, f2.y * cfac);
                }
            }
            if (r == 0) V4_TR(k, 14, 0);
            V4_WAIT(&bar_tile_done, (uint32_t)(k & 1));  // every P V and phi(K~)^T V of the block
            __syncwarp();
            tc_fence_after();
            if (r == 0) V4_TR(k, 14, 1);
            if (T.linear) {
                // Hc = Htot - Hsel, row f = r, as the MN-major B tile [c half 2][f 128][64 c] (bf16) in the
                // block's Hc slot; c phi(Q)_r over the block's Q buffer (its Q K^T are all done)
                V4_WAIT(&bar_v_full[gv_hc % NV], (uint32_t)((gv_hc / NV) & 1));  // the Hc slot is ours
                const uint32_t hb = sbase + OFF_V + (uint32_t)(gv_hc % NV) * VS_BYTES;
#pragma unroll
                for (int c0 = 0; c0 < 128; c0 += 32) {
                    uint32_t hs[32];
                    tmem_ld32(tmem + lane_base + TM_H + c0, hs);
                    tmem_ld_wait();
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        const int c = c0 + ch * 8;
                        const uint32_t* t8 = reinterpret_cast<const uint32_t*>(&htr[c >> 3]);
                        uint32_t o4[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 tf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t8[e]));
                            o4[e] = pack_bf16(tf.x - __uint_as_float(hs[ch * 8 + 2 * e]),
                                              tf.y - __uint_as_float(hs[ch * 8 + 2 * e + 1]));
                        }
                        st_shared_v4(hb + (c >> 6) * 16384 + sw128_off(r, c & 63), o4[0], o4[1], o4[2], o4[3]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_h_free);  // Hsel read: the next block's Hsel may start
                const uint32_t qb = sbase + OFF_Q + (uint32_t)b * Q_BYTES;
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {
                    const int c = ch * 8;
                    st_shared_v4(qb + (c >> 6) * 16384 + sw128_off(r, c & 63), cq[ch * 4], cq[ch * 4 + 1],
                                 cq[ch * 4 + 2], cq[ch * 4 + 3]);
                }
                fence_proxy_async_smem();  // Hc and c phi(Q) are read by the tensor core
            } else {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_h_free);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_lin_ready);
            if (r == 0) V4_TR(k, 14, 2);
            V4_WAIT(&bar_lin_done, (uint32_t)(k & 1));
            __syncwarp();
            tc_fence_after();
            if (r == 0) V4_TR(k, 14, 3);
            // out = alpha / l (O + (c phi(Q)) Hc), row r straight to global
            const float s_o = alpha / l;
            const uint32_t tO = tmem + lane_base + TM_O + (uint32_t)b * 128;
            uint4* orow = reinterpret_cast<uint4*>(p.out + grow * D);
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tO + c0, o);
                tmem_ld_wait();
                if (c0 == 96) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bar_o_free[b]);  // O(b) may take query block k + 2
                    if (r == 0) V4_TR(k, 14, 4);
                }
                if (live) {
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch)
                        orow[c0 / 8 + ch] = make_uint4(
                            pack_bf16(__uint_as_float(o[ch * 8 + 0]) * s_o, __uint_as_float(o[ch * 8 + 1]) * s_o),
                            pack_bf16(__uint_as_float(o[ch * 8 + 2]) * s_o, __uint_as_float(o[ch * 8 + 3]) * s_o),
                            pack_bf16(__uint_as_float(o[ch * 8 + 4]) * s_o, __uint_as_float(o[ch * 8 + 5]) * s_o),
                            pack_bf16(__uint_as_float(o[ch * 8 + 6]) * s_o, __uint_as_float(o[ch * 8 + 7]) * s_o));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

bool sparse_v4_eligible(const SparseLaunch& a) {
    return !a.dense && a.bq == 128 && a.bk == 64 && a.d == 128 && a.o_s == nullptr && a.o_l == nullptr &&
           a.big_l == nullptr && a.h_blocks == nullptr && a.z_blocks == nullptr && a.phiq != nullptr;
}

cudaError_t launch_sparse_v4(const SparseLaunch& a, cudaStream_t st, int* launches) {
    SparseV4Params p;
    p.kv_idx = a.kv_idx;
    p.kv_cnt = a.kv_cnt;
    p.kstride = a.kstride;
    p.kappa = a.kappa;
    p.rho = a.rho;
    p.ztot = a.ztot;
    p.zblk = a.zblk;
    p.htot16 = (const __nv_bfloat16*)a.htot16;
    p.phiq = (const __nv_bfloat16*)a.phiq;
    p.out = (__nv_bfloat16*)a.out;
    p.N = a.N;
    p.H = (int)a.H;
    p.tm = a.tm;
    p.tn = a.tn;
    p.ntiles = (int)(a.B * a.H) * a.tm;
    p.last_valid = a.N - (a.tn - 1) * v4::BK;
    p.scale_log2 = a.inv_sqrt_d * 1.4426950408889634f;
#ifdef SLA2_TRACE
    extern unsigned long long* g_trace_buf;
    p.trace = g_trace_buf;
#endif
    cudaError_t e = ensure_smem_attr((const void*)sla2_sparse_v4_kernel, (int)v4::SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = p.ntiles < sms ? p.ntiles : sms;
    sla2_sparse_v4_kernel<<<grid, v4::NTHREADS, v4::SMEM, st>>>(*a.tm_q, *a.tm_k, *a.tm_v, *a.tm_phik, p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
