// sparse_bf16.cu -- the SLA2 sparse + linear + alpha-blend forward for one (b, h, query block)
// per CTA, on tcgen05 tensor cores with TMEM accumulators and TMA gathers (sm_100a).
//
// Replaces the per-query-block loop of sla2_forward_blockwise (attention.hpp:484-558) and its
// helpers block_scores_qk / block_product_pv (attention.hpp:372-415), for bq = 128, bk = 64,
// d = 128 (the paper's blocks), bf16 operands, fp32 accumulation.
//
// Per CTA (query block i of head bh, kept key blocks j_0 < j_1 < ... from the router), key
// blocks are processed in PAIRS (2p, 2p+1) in ascending order:
//   S_pair = Q_i [K_2p; K_2p+1]^T          tcgen05 kind::f16 SS, M128 N128 K128 -> TMEM (2 pair buffers)
//   P      = exp2(S*log2e/sqrt(d) - m)      softmax warps, lazily rescaled running max; P is
//                                           written back over each block's S in TMEM as bf16
//   O     += P_j V_j                        TS: P from TMEM, V_j from smem, M128 N128 K64
//   Hsel  += phi(K~_j)^T V_j                SS, M128 N128 K64 (MN-major A and B)
// epilogue (fused, attention.hpp:532-557):
//   O_s = O / l
//   Hc  = Htot - Hsel, Zc = Ztot - sum_sel z_j      ("total minus selected" = the
//                                                    reference's complement sum, 495-502)
//   O_l = (phi(Q) Hc) / (phi(Q) . Zc)              SS, M128 N128 K128
//   out = alpha O_s + (1 - alpha) O_l, alpha = sigmoid(rho_i) (forced to 1 on full rows)
// The raw K is used for Q K^T: smoothing shifts every score of a row by the same constant
// (test_attention.cpp:270-279), so O_s is unchanged and K needs no bf16 re-rounding.
//
// Why pairs: on B200 a kind::f16 M128 tcgen05.mma costs max(~96, N/2) cycles
// (tools/umma_bench.py), so Q K^T over one 64-key block (N = 64) runs at a third of the
// tensor rate; two blocks per instruction (N = 128) halve the QK instruction count.
//
// Warp roles (256 threads, 1 CTA/SM): w0 TMA producer (Q, K pair ring, then phi(Q) over Q once
// the last Q K^T has read Q), w1 MMA issuer, w2 TMEM allocator + TMA producer (V / phi(K) ring,
// Htot), w3 Zc; then w0, w2, w3 together form the denominators phi(Q) . Zc, w4-7 softmax /
// correction / epilogue (thread = query row). phi(Q) itself is computed on the router's query
// side (launch_phiq), off the critical path, and arrives by TMA.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

namespace sp {
constexpr int BQ = 128, BK = 64, D = 128;
constexpr int NKP = 2, NSV = 4;  // K pair ring (32 KB/stage), V+phi(K) ring (32 KB/stage)
constexpr uint32_t Q_BYTES = BQ * D * 2;     // 32 KB
constexpr uint32_t TILE_BYTES = BK * D * 2;  // 16 KB (one K, V or phi(K) tile)
constexpr uint32_t KP_BYTES = 2 * TILE_BYTES;  // K pair: [k_atom 2][128 rows][128 B]
constexpr uint32_t HT_BYTES = D * D * 2;     // 32 KB Htot (bf16), staged in a free V stage
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
constexpr uint32_t OFF_V = OFF_K + NKP * KP_BYTES;
constexpr uint32_t SMEM_BYTES = OFF_V + NSV * 2 * TILE_BYTES;  // 224 KB
constexpr uint32_t SMEM_ALLOC = SMEM_BYTES + 1024;
// TMEM columns (512 allocated)
constexpr uint32_t TM_S = 0;    // 128: S fp32 of the current pair (block 2p in cols 0-63, 2p+1 in 64-127)
constexpr uint32_t TM_P = 128;  // 2 x 64: P bf16 of pairs n & 1 (block 2p in the first 32, 2p+1 next)
constexpr uint32_t TM_O = 256;  // 128: O accumulator
constexpr uint32_t TM_H = 384;  // 128: Hsel accumulator
constexpr uint32_t TM_L = 0;    // 128: phi(Q) Hc after the loop (the S columns are free then)
constexpr float RESCALE_LOG2 = 8.0f;  // lazy rescale threshold (P <= 2^8)
}  // namespace sp

struct SparseBf16Params {
    const int32_t* kv_idx;
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* rho;
    const float* ztot;
    const float* zblk;
    const float* mu;
    const __nv_bfloat16* q;
    __nv_bfloat16* out;
    float* o_s;
    float* o_l;
    float* big_l;
    float* h_blocks;
    float* z_blocks;
    const float* htot32;
    int N, H, tm, tn;
    int last_valid;  // keys in the last key block (BK unless N % BK != 0)
    float scale_log2;
    float inv_sqrt_d;
    int dense;
#ifdef SLA2_TRACE
    unsigned long long* trace;
#endif
};

#ifdef SLA2_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SLA2_TR(slot) p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 128 + (slot)] = gtimer()
#else
#define SLA2_TR(slot)
#endif

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// den[r] = phi(Q)_r . Zc for query row r, from the bf16 phi(Q) tile (the A operand of the final
// MMA, so numerator and denominator see the same rounded phi(Q)); four partial sums.
__device__ __forceinline__ void den_row(uint32_t qb, int r, const float* sZc, float* sDen) {
    float d4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ch = 0; ch < 16; ++ch) {
        uint32_t w[4];
        ld_shared_v4(qb + (ch >> 3) * 16384 + sw128_off(r, (ch & 7) * 8), w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
            const int f = ch * 8 + 2 * e;
            d4[e] = fmaf(f2.y, sZc[f + 1], fmaf(f2.x, sZc[f], d4[e]));
        }
    }
    sDen[r] = (d4[0] + d4[1]) + (d4[2] + d4[3]);
}

__global__ void __launch_bounds__(256, 1)
    sla2_sparse_bf16_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmPhi,
                            const __grid_constant__ CUtensorMap tmHt, const __grid_constant__ CUtensorMap tmPq,
                            const __grid_constant__ CUtensorMap tmO, const SparseBf16Params p) {
    using namespace sp;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_q, bar_qt, bar_qk_done, bar_mma_done, bar_pq, bar_zc, bar_ht, bar_k_full[NKP],
        bar_k_empty[NKP],
        bar_v_full[NSV],
        bar_v_empty[NSV], bar_s_full, bar_s_free, bar_p_full[2], bar_pv_done[2], bar_lin_ready, bar_lin_done;
    __shared__ uint32_t tmem_base_sh;
    __shared__ float sZc[D];
    __shared__ float sDen[BQ];
    __shared__ float sInvL[BQ];  // 1 / l per row, for the 8-warp epilogue

    const int i = blockIdx.x;       // query block
    const int64_t bh = blockIdx.y;  // (b, h)
    const int h = (int)(bh % p.H);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool dense = p.dense != 0;
    const int nb = dense ? p.tn : (p.kv_cnt ? p.kv_cnt[bh * p.tm + i] : p.kappa);
    const int npair = (nb + 1) >> 1;
    const int32_t* idx = p.kv_idx + (bh * p.tm + i) * (int64_t)p.kstride;
    const bool full_row = dense || (nb == p.tn);
    const bool linear = !full_row;

    uint8_t* sQ = smem + OFF_Q;
    auto sKp = [&](int s) { return smem + OFF_K + s * KP_BYTES; };
    auto sV = [&](int s) { return smem + OFF_V + s * 2 * TILE_BYTES; };
    auto sPh = [&](int s) { return smem + OFF_V + s * 2 * TILE_BYTES + TILE_BYTES; };
    auto kblock = [&](int j) { return dense ? j : idx[j]; };
    const uint32_t v_tx = dense ? TILE_BYTES : 2 * TILE_BYTES;  // V (+ phi(K~)) per stage
    constexpr int NV0 = 2;  // V stages thread 0 fills before the CTA-wide barrier

    if (threadIdx.x == 0) {
        // the kept-block indices of the first pair: their global loads overlap the barrier setup
        int jk[2] = {kblock(0), nb > 1 ? kblock(1) : 0};
        mbar_init(&bar_q, 1);
        mbar_init(&bar_qt, 128);  // Q copied into TMEM by the softmax warps
        mbar_init(&bar_qk_done, 1);
        mbar_init(&bar_mma_done, 1);
        mbar_init(&bar_pq, 1);
        mbar_init(&bar_zc, 1);
        mbar_init(&bar_ht, 1);
        for (int s = 0; s < NKP; ++s) {
            mbar_init(&bar_k_full[s], 1);
            mbar_init(&bar_k_empty[s], 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(&bar_v_full[s], 1);
            mbar_init(&bar_v_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_p_full[b], 128);
            mbar_init(&bar_pv_done[b], 1);
        }
        mbar_init(&bar_s_full, 1);
        mbar_init(&bar_s_free, 128);
        mbar_init(&bar_lin_ready, 256);
        mbar_init(&bar_lin_done, 1);
        fence_barrier_init();
        // Q, the first K pair and the first V / phi(K~) stages go out before the TMEM allocation
        // and the CTA barrier (they need only the initialized mbarriers): ~0.5 us off the prologue
        const int qrow = i * BQ, hz = (int)bh;
        const uint64_t pol_keep = policy_evict_last();
        mbar_arrive_expect_tx(&bar_q, Q_BYTES);
        tma_load_3d(sQ, &tmQ, 0, qrow, hz, &bar_q);
        tma_load_3d(sQ + 8192, &tmQ, 0, qrow + 64, hz, &bar_q);
        tma_load_3d(sQ + 16384, &tmQ, 64, qrow, hz, &bar_q);
        tma_load_3d(sQ + 24576, &tmQ, 64, qrow + 64, hz, &bar_q);
        const int cnt0 = min(2, nb);
        mbar_arrive_expect_tx(&bar_k_full[0], cnt0 * TILE_BYTES);
        for (int b = 0; b < cnt0; ++b) {
            tma_load_3d_hint(sKp(0) + b * 8192, &tmK, 0, jk[b] * BK, hz, &bar_k_full[0], pol_keep);
            tma_load_3d_hint(sKp(0) + 16384 + b * 8192, &tmK, 64, jk[b] * BK, hz, &bar_k_full[0], pol_keep);
        }
        for (int j = 0; j < NV0 && j < nb; ++j) {
            mbar_arrive_expect_tx(&bar_v_full[j], v_tx);
            tma_load_3d_hint(sV(j), &tmV, 0, jk[j] * BK, hz, &bar_v_full[j], pol_keep);
            tma_load_3d_hint(sV(j) + 8192, &tmV, 64, jk[j] * BK, hz, &bar_v_full[j], pol_keep);
            if (!dense) {
                tma_load_3d_hint(sPh(j), &tmPhi, 0, jk[j] * BK, hz, &bar_v_full[j], pol_keep);
                tma_load_3d_hint(sPh(j) + 8192, &tmPhi, 64, jk[j] * BK, hz, &bar_v_full[j], pol_keep);
            }
        }
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (threadIdx.x == 0) SLA2_TR(0);

    // epilogue buffers in V stages: Htot goes where block nb would have gone (loaded by the V
    // producer once that stage drains), Hc into the next one (free once every PV is done)
    uint8_t* sHt = sV(nb % NSV);
    uint8_t* sHc = sV((nb + 1) % NSV);

    if (warp == 0) {
        // ===================== TMA producer: Q, K pair ring =====================
        if (lane == 0) {
            tma_prefetch_desc(&tmQ);
            tma_prefetch_desc(&tmK);
            const uint64_t pol_keep = policy_evict_last();
            const int qrow = i * BQ, hz = (int)bh;  // 3-D maps: (column, row in head, head)
            // Q and pair 0 were issued by this thread before the CTA barrier
            for (int n = 1; n < npair; ++n) {
                const int s = n % NKP;
                if (n >= NKP) mbar_wait(&bar_k_empty[s], ((n / NKP) - 1) & 1);
                const int cnt = min(2, nb - 2 * n);
                if (n == 0) SLA2_TR(54);
                if (n == npair - 1) SLA2_TR(55);
                mbar_arrive_expect_tx(&bar_k_full[s], cnt * TILE_BYTES);
                for (int b = 0; b < cnt; ++b) {
                    const int krow = kblock(2 * n + b) * BK;
                    // rows b*64.. of each 128-row k-atom: [cols 0-63] then [cols 64-127]
                    tma_load_3d_hint(sKp(s) + b * 8192, &tmK, 0, krow, hz, &bar_k_full[s], pol_keep);
                    tma_load_3d_hint(sKp(s) + 16384 + b * 8192, &tmK, 64, krow, hz, &bar_k_full[s], pol_keep);
                }
            }
            if (linear) {
                // phi(Q) over Q once nothing reads Q from shared memory any more (same layout)
                tma_prefetch_desc(&tmPq);
                mbar_wait(&bar_qk_done, 0);
                mbar_arrive_expect_tx(&bar_pq, Q_BYTES);
                tma_load_3d(sQ, &tmPq, 0, qrow, hz, &bar_pq);
                tma_load_3d(sQ + 8192, &tmPq, 0, qrow + 64, hz, &bar_pq);
                tma_load_3d(sQ + 16384, &tmPq, 64, qrow, hz, &bar_pq);
                tma_load_3d(sQ + 24576, &tmPq, 64, qrow + 64, hz, &bar_pq);
            }
        }
    } else if (warp == 2) {
        // ===================== TMA producer: V / phi(K) ring, Htot =====================
        if (lane == 0) {
            tma_prefetch_desc(&tmV);
            if (!dense) tma_prefetch_desc(&tmPhi);
            const uint64_t pol_keep = policy_evict_last();
            const bool ldphi = !dense;
            const uint32_t tx = ldphi ? 2 * TILE_BYTES : TILE_BYTES;
            // stages 0 .. NV0-1 were issued by thread 0 before the CTA barrier (with phi(K~) unless
            // dense; the SLA2_EXP_NOPHIK experiment loads V only from stage NV0 on)
            for (int j = NV0; j < nb; ++j) {
                const int s = j % NSV;
                if (j >= NSV) mbar_wait(&bar_v_empty[s], ((j / NSV) - 1) & 1);
                const int krow = kblock(j) * BK, hz = (int)bh;
                if (j < 16) SLA2_TR(64 + j);
                mbar_arrive_expect_tx(&bar_v_full[s], tx);
                tma_load_3d_hint(sV(s), &tmV, 0, krow, hz, &bar_v_full[s], pol_keep);
                tma_load_3d_hint(sV(s) + 8192, &tmV, 64, krow, hz, &bar_v_full[s], pol_keep);
                if (ldphi) {
                    tma_load_3d_hint(sPh(s), &tmPhi, 0, krow, hz, &bar_v_full[s], pol_keep);
                    tma_load_3d_hint(sPh(s) + 8192, &tmPhi, 64, krow, hz, &bar_v_full[s], pol_keep);
                }
            }
            if (linear) {
                // Htot of this head, bf16 [f][c] as the MN-major B layout [c_atom][f][64], into the
                // stage block nb would use (same wait rule as a V load)
                const int s = nb % NSV;
                if (nb >= NSV) mbar_wait(&bar_v_empty[s], ((nb / NSV) - 1) & 1);
                tma_prefetch_desc(&tmHt);
                mbar_arrive_expect_tx(&bar_ht, HT_BYTES);
                tma_load_2d_hint(sHt, &tmHt, 0, (int)(bh * D), &bar_ht, pol_keep);
                tma_load_2d_hint(sHt + 16384, &tmHt, 64, (int)(bh * D), &bar_ht, pol_keep);
            }
        }
#ifdef SLA2_TRACE
        else if (lane == 1) {
            // trace only: stamp each V/phi(K) stage's actual arrival
            for (int j = 0; j < nb && j < 16; ++j) {
                for (int it = 0; it < 1000000 && !mbar_try_wait(&bar_v_full[j % NSV], (j / NSV) & 1); ++it) {
                }
                SLA2_TR(96 + j);
            }
        }
#endif
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, elect.sync issues) =====================
        // All 32 lanes run this with warp-uniform values (counts and TMEM base via shfl), so
        // the descriptors live in uniform registers and each MMA is a few instructions.
        constexpr uint32_t ID_QK2 = idesc_bf16(128, 128, false, false);
        constexpr uint32_t ID_QK1 = idesc_bf16(128, 64, false, false);
        constexpr uint32_t ID_PV = idesc_bf16(128, 128, false, true);
        constexpr uint32_t ID_HS = idesc_bf16(128, 128, true, true);
        const uint32_t tm = warp_uniform(tmem);
        const int nbu = (int)warp_uniform((uint32_t)nb);
        const int npu = (nbu + 1) >> 1;
        const uint32_t sbase = warp_uniform(smem_u32(smem));
        // descriptor bases; + (byte offset >> 4) advances the start address
        const uint64_t dQ = sdesc_sw128(sbase + OFF_Q, 16, 1024);
        const uint64_t dK0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
        const uint64_t dVm = sdesc_sw128(sbase + OFF_V, 8192, 1024);  // MN-major V / phi(K) tiles
        mbar_wait(&bar_q, 0);
        tc_fence_after();
        if (lane == 0) SLA2_TR(1);
        // Static issue order (the tensor pipe runs MMAs in issue order):
        //   QK(0); for each pair n: [S(n) read] QK(n+1); [P(n)] PV(n), HS(n)
        // S has one buffer and P its own two, so QK(n+1) enters the pipe as soon as the softmax
        // has loaded S(n) into registers and runs under the softmax of pair n; PV(n) and HS(n)
        // run under the softmax of pair n+1.
        auto issue_qk = [&](int n) {
            const int s = n % NKP;
            mbar_wait(&bar_k_full[s], (n / NKP) & 1);
            tc_fence_after();
            if (lane == 0 && n < 8) SLA2_TR(56 + n);
            const uint32_t idq = (2 * n + 1 < nbu) ? ID_QK2 : ID_QK1;
            const uint64_t dK = dK0 + ((s * KP_BYTES) >> 4);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint32_t off = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
                umma_bf16_ss_w(tm + TM_S, dQ + off, dK + off, idq, ks > 0);
            }
            umma_commit_w(&bar_s_full);
            umma_commit_w(&bar_k_empty[s]);
            if (n == npu - 1) umma_commit_w(&bar_qk_done);
        };
        if (npu > 0) issue_qk(0);
        for (int n = 0; n < npu; ++n) {
            const int j0 = 2 * n, j1 = min(nbu, j0 + 2);
            if (n + 1 < npu) {
                mbar_wait(&bar_s_free, n & 1);  // the softmax holds S(n) in registers
                tc_fence_after();
                issue_qk(n + 1);
            }
            mbar_wait(&bar_p_full[n & 1], (n >> 1) & 1);
            tc_fence_after();
            // PV(n), then HS(n) (the V/phi(K) stages are released after it).
            // (Interleaving PV and HS k-steps measured slower: 1.50 vs 1.28 us per pair.)
            for (int j = j0; j < j1; ++j) {
                const int sv = j % NSV;
                mbar_wait(&bar_v_full[sv], (j / NSV) & 1);
                tc_fence_after();
                if (lane == 0 && j < 16) SLA2_TR(80 + j);
                const uint64_t dV = dVm + ((sv * 2 * TILE_BYTES) >> 4);
                const uint32_t aP = tm + TM_P + (n & 1) * 64 + (j & 1) * 32;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    umma_bf16_ts_w(tm + TM_O, aP + ks * 8, dV + ((ks * 2048) >> 4), ID_PV, (j > 0 || ks > 0));
                if (dense) umma_commit_w(&bar_v_empty[sv]);
            }
            umma_commit_w(&bar_pv_done[n & 1]);
            if (lane == 0 && n < 16) SLA2_TR(34 + n);
            if (!dense) {
                for (int j = j0; j < j1; ++j) {
                    const int sv = j % NSV;
                    const uint64_t dV = dVm + ((sv * 2 * TILE_BYTES) >> 4);
                    const uint64_t dP = dV + (TILE_BYTES >> 4);  // phi(K) tile follows V in the stage
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        umma_bf16_ss_w(tm + TM_H, dP + ((ks * 2048) >> 4), dV + ((ks * 2048) >> 4), ID_HS,
                                       (j > 0 || ks > 0));
                    umma_commit_w(&bar_v_empty[sv]);  // after PV_j and HS_j
                }
            }
            if (lane == 0 && n < 16) SLA2_TR(112 + n);
        }
        umma_commit_w(&bar_mma_done);  // every QK / PV / HS of the loop
    } else if (warp == 3) {
        // ===================== Zc, then phi(Q) in place over sQ and phi(Q) . Zc =====================
        if (linear) {
            // lane owns features 4*lane .. 4*lane+3; one coalesced 512-B row per kept block
            const float* zb = p.zblk + bh * (int64_t)p.tn * D + lane * 4;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j0 = 0; j0 < nb; j0 += 32) {
                const int myj = (j0 + lane < nb) ? idx[j0 + lane] : 0;
                const int cnt = min(32, nb - j0);
                int u = 0;
                for (; u + 4 <= cnt; u += 4) {
                    float4 z[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        z[t] = *reinterpret_cast<const float4*>(zb + (int64_t)__shfl_sync(0xffffffffu, myj, u + t) * D);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        acc.x += z[t].x;
                        acc.y += z[t].y;
                        acc.z += z[t].z;
                        acc.w += z[t].w;
                    }
                }
                for (; u < cnt; ++u) {
                    const float4 z = *reinterpret_cast<const float4*>(zb + (int64_t)__shfl_sync(0xffffffffu, myj, u) * D);
                    acc.x += z.x;
                    acc.y += z.y;
                    acc.z += z.z;
                    acc.w += z.w;
                }
            }
            const float4 zt = *reinterpret_cast<const float4*>(p.ztot + bh * D + lane * 4);
            sZc[lane * 4 + 0] = zt.x - acc.x;
            sZc[lane * 4 + 1] = zt.y - acc.y;
            sZc[lane * 4 + 2] = zt.z - acc.z;
            sZc[lane * 4 + 3] = zt.w - acc.w;
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_zc);
        }
        if (p.z_blocks) {  // SLA2ForwardSaved z_blocks (zero on full rows)
            const float4 z = linear ? make_float4(sZc[lane * 4], sZc[lane * 4 + 1], sZc[lane * 4 + 2], sZc[lane * 4 + 3])
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(p.z_blocks + (bh * p.tm + i) * D + lane * 4) = z;
        }
    } else if (warp >= 4) {
        // ===================== softmax / correction / epilogue =====================
        const int r = threadIdx.x - 128;  // query row within the block
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const float rho_i = linear ? p.rho[(int64_t)h * p.tm + i] : 0.0f;  // loaded now, used after the loop
        // ragged N: does this row keep the partial last key block? (one load, before the loop)
        const bool tail_kept = p.last_valid < BK && kblock(nb - 1) == p.tn - 1;
        float m2 = -INFINITY, l = 0.0f;
        for (int n = 0; n < npair; ++n) {
            const int b = n & 1;
            const bool two = 2 * n + 1 < nb;
            mbar_wait(&bar_s_full, n & 1);
            __syncwarp();
            if (r == 0 && n < 16) SLA2_TR(2 + n);
            tc_fence_after();
            const uint32_t sbase = tmem + lane_base + TM_S;
            if (tail_kept && n == npair - 1) {
                // ragged N: keys past N in the partial last key block (zero-filled K) get -inf,
                // written into S in TMEM before the load (no extra registers in the softmax).
                // Kept blocks ascend, so that block is the row's last one (nb - 1).
                const uint32_t col0 = (uint32_t)(((nb - 1) - 2 * n) * 64);
                for (int t = p.last_valid; t < BK; ++t) tmem_st1(sbase + col0 + t, __float_as_uint(-INFINITY));
                tmem_st_wait();
            }
            uint32_t sr[128];
            tmem_ld32(sbase, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
            tmem_ld32(sbase + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
            if (two) {
                tmem_ld32(sbase + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
                tmem_ld32(sbase + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
            }
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&bar_s_free);  // QK(n+1) may overwrite S now
            // row max as four independent FMNMX3 chains (one 64-long chain was ~0.13 us a pair)
            float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int t = 0; t < 64; t += 8) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    m4[u] = fmaxf(m4[u], fmaxf(__uint_as_float(sr[t + 2 * u]), __uint_as_float(sr[t + 2 * u + 1])));
            }
            if (two) {
#pragma unroll
                for (int t = 64; t < 128; t += 8) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        m4[u] = fmaxf(m4[u], fmaxf(__uint_as_float(sr[t + 2 * u]), __uint_as_float(sr[t + 2 * u + 1])));
                }
            }
            float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
            mx *= p.scale_log2;
            if (n == 0) {
                m2 = mx;
            } else {
                const bool need = mx > m2 + RESCALE_LOG2;
                if (__any_sync(0xffffffffu, need)) {
                    const float mnew = fmaxf(m2, mx);
                    const float corr = fast_exp2(m2 - mnew);
                    mbar_wait(&bar_pv_done[(n - 1) & 1], ((n - 1) >> 1) & 1);  // all PVs so far done
                    __syncwarp();
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 128; c0 += 32) {
                        uint32_t o[32];
                        tmem_ld32(tmem + lane_base + TM_O + c0, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st32(tmem + lane_base + TM_O + c0, o);
                    }
                    l *= corr;
                    m2 = mnew;
                }
            }
            // P = exp2(s * scale - m2) as packed bf16 into P buffer n & 1, last read by PV(n-2)
            if (n >= 2) {
                mbar_wait(&bar_pv_done[b], ((n - 2) >> 1) & 1);
                __syncwarp();
                tc_fence_after();
            }
            const uint32_t pbase = tmem + lane_base + TM_P + b * 64;
            float rs0 = 0.0f, rs1 = 0.0f;
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                if (blk == 1 && !two) break;
                uint32_t w[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float p0 = fast_exp2(fmaf(__uint_as_float(sr[blk * 64 + 2 * e]), p.scale_log2, -m2));
                    const float p1 = fast_exp2(fmaf(__uint_as_float(sr[blk * 64 + 2 * e + 1]), p.scale_log2, -m2));
                    rs0 += p0;
                    rs1 += p1;
                    w[e] = pack_bf16(p0, p1);
                }
                tmem_st32(pbase + blk * 32, w);
            }
            l += rs0 + rs1;
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&bar_p_full[b]);
            if (r == 0 && n < 16) SLA2_TR(18 + n);
        }
        // row statistics for the 8-warp epilogue (published through bar_lin_ready)
        sInvL[r] = 1.0f / l;
        if (linear) {  // den = phi(Q)_r . Zc, from the TMA-loaded phi(Q) tile
            mbar_wait(&bar_zc, 0);
            mbar_wait(&bar_pq, 0);
            den_row(smem_u32(sQ), r, sZc, sDen);
        }
        if (p.big_l && i * BQ + r < p.N) {
            // L with raw K scores, shifted to the smoothed-K scores the reference uses:
            // q_r . K~_t = q_r . K_t - q_r . mu
            const int64_t grow = bh * p.N + (int64_t)i * BQ + r;
            float shift = 0.0f;
            if (p.mu) {
                const float* mu = p.mu + bh * D;
                const __nv_bfloat16* qg = p.q + grow * D;
                for (int f = 0; f < D; ++f) shift += __bfloat162float(qg[f]) * mu[f];
                shift *= p.inv_sqrt_d;
            }
            p.big_l[grow] = m2 / 1.4426950408889634f + logf(l) - shift;
        }
    }

    // ===================== epilogue, all eight warps =====================
    // Warp w serves rows 32 (w % 4) + lane (its TMEM lane quarter) and column half
    // ch = w < 4 ? 1 : 0 of Hc and of the output, so each thread moves 64 columns, not 128.
    {
        __syncwarp();
        const int q4 = warp & 3, r = q4 * 32 + lane;
        const int c0 = warp < 4 ? 64 : 0;
        const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
        mbar_wait(&bar_mma_done, 0);  // every QK / PV / HS of the loop is complete
        __syncwarp();
        tc_fence_after();
        if (threadIdx.x == 128) SLA2_TR(50);
        float alpha = 1.0f;
        if (linear) {
            // alpha = sigmoid(rho_i) with the reference's clamp (attention.hpp:17-22)
            const float x = p.rho[(int64_t)h * p.tm + i];
            float a = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x)));
            a = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
            alpha = a;
            // Hc = Htot - Hsel: row f = r, columns c0 .. c0 + 63, bf16 into the MN-major B tile
            mbar_wait(&bar_ht, 0);
            __syncwarp();
            const uint32_t hb = smem_u32(sHc), htb = smem_u32(sHt);
            uint32_t hs[64];
            tmem_ld32(tmem + lane_base + TM_H + c0, *reinterpret_cast<uint32_t(*)[32]>(&hs[0]));
            tmem_ld32(tmem + lane_base + TM_H + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&hs[32]));
            tmem_ld_wait();
            if (p.h_blocks) {  // SLA2ForwardSaved h_blocks: fp32 Htot - Hsel, row f = r
                const float* ht = p.htot32 + bh * D * D + r * D + c0;
                float* hb_out = p.h_blocks + ((bh * p.tm + i) * D + r) * D + c0;
                for (int c = 0; c < 64; ++c) hb_out[c] = ht[c] - __uint_as_float(hs[c]);
            }
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                const uint32_t off = (c0 >> 6) * 16384 + sw128_off(r, ch * 8);
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
            fence_proxy_async_smem();
            tc_fence_before();
        }
        if (!linear && p.h_blocks) {  // full row: the complement is empty (attention.hpp:495)
            float* hb_out = p.h_blocks + ((bh * p.tm + i) * D + r) * D + c0;
            for (int c = 0; c < 64; ++c) hb_out[c] = 0.0f;
        }
        mbar_arrive(&bar_lin_ready);  // also publishes sInvL (written by the softmax warps)
        mbar_wait(&bar_lin_ready, 0);
        if (threadIdx.x == 128) SLA2_TR(51);
        if (linear && warp == 1) {
            // O_l numerator = phi(Q) (Htot - Hsel): A = phi(Q) (K-major, in sQ), B = Hc (MN-major)
            mbar_wait(&bar_pq, 0);
            tc_fence_after();
            constexpr uint32_t ID_LIN = idesc_bf16(128, 128, false, true);
            const uint32_t tm = warp_uniform(tmem);
            const uint64_t dQl = sdesc_sw128(warp_uniform(smem_u32(sQ)), 16, 1024);
            const uint64_t dH = sdesc_sw128(warp_uniform(smem_u32(sHc)), 16384, 1024);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint32_t off = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
                umma_bf16_ss_w(tm + TM_L, dQl + off, dH + ((ks * 2048) >> 4), ID_LIN, ks > 0);
            }
            umma_commit_w(&bar_lin_done);
        }
        float inv_den = 0.0f;
        if (linear) {
            inv_den = 1.0f / sDen[r];  // written before bar_lin_ready by the softmax warps
            mbar_wait(&bar_lin_done, 0);
            __syncwarp();
            tc_fence_after();
        }
        if (threadIdx.x == 128) SLA2_TR(52);
        // out = alpha * O / l + (1 - alpha) * num / den, columns c0 .. c0 + 63 of row r
        const float inv_l = sInvL[r];
        const float beta = 1.0f - alpha;
        const int64_t grow = bh * p.N + (int64_t)i * BQ + r;
        const bool want_saved = p.o_s != nullptr && i * BQ + r < p.N;  // ragged tail: not stored
        const uint32_t ob = smem_u32(sQ);  // every MMA reading sQ (Q K^T, phi(Q) Hc) is complete
        uint32_t o[64], ln[64];
        tmem_ld32(tmem + lane_base + TM_O + c0, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
        tmem_ld32(tmem + lane_base + TM_O + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
        if (linear) {
            tmem_ld32(tmem + lane_base + TM_L + c0, *reinterpret_cast<uint32_t(*)[32]>(&ln[0]));
            tmem_ld32(tmem + lane_base + TM_L + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&ln[32]));
        }
        tmem_ld_wait();
        float res[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) {
            const float os = __uint_as_float(o[c]) * inv_l;
            const float ol = linear ? __uint_as_float(ln[c]) * inv_den : 0.0f;
            res[c] = linear ? alpha * os + beta * ol : os;
            if (want_saved) {
                p.o_s[grow * D + c0 + c] = os;
                p.o_l[grow * D + c0 + c] = ol;
            }
        }
        // bf16 half-row into the (now free) Q tile, SW128 layout: one TMA store writes the block
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
            st_shared_v4(ob + (c0 >> 6) * 16384 + sw128_off(r, ch * 8), pack_bf16(res[ch * 8 + 0], res[ch * 8 + 1]),
                         pack_bf16(res[ch * 8 + 2], res[ch * 8 + 3]), pack_bf16(res[ch * 8 + 4], res[ch * 8 + 5]),
                         pack_bf16(res[ch * 8 + 6], res[ch * 8 + 7]));
        fence_proxy_async_smem();
        tc_fence_before();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int orow0 = i * BQ, hz = (int)bh;  // rows past N (ragged tail) are dropped
        tma_store_3d(&tmO, 0, orow0, hz, sQ);
        tma_store_3d(&tmO, 0, orow0 + 64, hz, sQ + 8192);
        tma_store_3d(&tmO, 64, orow0, hz, sQ + 16384);
        tma_store_3d(&tmO, 64, orow0 + 64, hz, sQ + 24576);
        tma_store_commit();
        SLA2_TR(53);
        tma_store_wait_read();  // sQ must stay valid until the store has read it
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

#ifdef SLA2_TRACE
unsigned long long* g_trace_buf = nullptr;
extern "C" void sla2_trace_set_buffer(unsigned long long* b) { g_trace_buf = b; }
#endif

cudaError_t launch_sparse_bf16(const SparseLaunch& a, cudaStream_t st, int* launches) {
    SparseBf16Params p;
    p.kv_idx = a.kv_idx;
    p.kv_cnt = a.kv_cnt;
    p.kstride = a.kstride;
    p.kappa = a.kappa;
    p.rho = a.rho;
    p.ztot = a.ztot;
    p.zblk = a.zblk;
    p.mu = a.smooth ? a.mu : nullptr;
    p.q = (const __nv_bfloat16*)a.q;
    p.out = (__nv_bfloat16*)a.out;
    p.o_s = a.o_s;
    p.o_l = a.o_l;
    p.big_l = a.big_l;
    p.h_blocks = a.dense ? nullptr : a.h_blocks;
    p.z_blocks = a.dense ? nullptr : a.z_blocks;
    p.htot32 = a.htot;
    p.N = a.N;
    p.H = (int)a.H;
    p.tm = a.tm;
    p.tn = a.tn;
    p.last_valid = a.N - (a.tn - 1) * sp::BK;
    p.inv_sqrt_d = a.inv_sqrt_d;
    p.scale_log2 = a.inv_sqrt_d * 1.4426950408889634f;
    p.dense = a.dense;
#ifdef SLA2_TRACE
    p.trace = g_trace_buf;
#endif
    ensure_smem_attr((const void*)sla2_sparse_bf16_kernel, (int)(sp::SMEM_ALLOC));
    if (a.o_s == nullptr && a.o_l != nullptr) return cudaErrorInvalidValue;
    dim3 grid(a.tm, (unsigned)(a.B * a.H));
    if ((!a.dense && !a.tm_phiq) || !a.tm_out) return cudaErrorInvalidValue;
    sla2_sparse_bf16_kernel<<<grid, 256, sp::SMEM_ALLOC, st>>>(*a.tm_q, *a.tm_k, *a.tm_v,
                                                                a.dense ? *a.tm_k : *a.tm_phik,
                                                                a.dense ? *a.tm_k : *a.tm_ht,
                                                                a.dense ? *a.tm_k : *a.tm_phiq, *a.tm_out, p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
