// sparse_fa.cu -- the SLA2 sparse forward as two sm_100a kernels (bf16, d = 128, bq = 128, bk = 64).
//
// The per-query-block loop of sla2_forward_blockwise (attention.hpp:484-558) has two branches
// that share the kept key blocks: the softmax branch over the kept blocks (block_scores_qk /
// block_product_pv, 372-415) and the linear branch over the complement (495-502). One CTA
// cannot hold both branches' accumulators for two query blocks at once: TMEM has 512 columns
// and S, O, Hsel take 128 each. With one query block per CTA the softmax runs on one warp per
// SM sub-partition and cannot keep the tensor pipe busy (profiles/trace_v2_r02.txt: ~1.1 us of
// softmax per key-block pair against ~0.8 us of tensor work). So the forward is split:
//
//  * sla2_linsel_kernel: per query block i, Hsel = sum_sel phi(K~_j)^T V_j on tcgen05 (TMEM),
//    Hc = Htot - Hsel, O_l = phi(Q_i) Hc / (phi(Q_i) . Zc), Zc = Ztot - sum_sel z_j, written to
//    HBM as bf16. Persistent: the (V_j, phi(K~_j)) ring runs across query blocks and Hsel is
//    double buffered in TMEM, so one block's epilogue overlaps the next one's loads and MMAs.
//  * sla2_attn_kernel: FlashAttention-style softmax branch with TWO query blocks per CTA
//    ("lanes" A and B), each with its own S / O accumulators in TMEM (S_A | O_A | S_B | O_B =
//    512 columns, P written as bf16 over S) and its own softmax warpgroup, so the tensor pipe
//    runs one lane's Q K^T / P V while the other lane's softmax works. A separate epilogue
//    warpgroup forms out = alpha O / l + (1 - alpha) O_l (attention.hpp:532-557) and frees O
//    for the lane's next query block. The same kernel with every key block kept and no linear
//    term is full_attention (attention.hpp:71-75), the dense baseline.
//
// Warp roles of sla2_attn_kernel (512 threads, one CTA per SM, persistent):
//   warps 0, 3  TMA producer of lane A / lane B: Q per query block (once the previous one's last
//               Q K^T is done), K and V per key block into the lane's own rings
//   warps 1, 2  MMA issuer of lane A / lane B: Q K^T(0), Q K^T(1), then per step the lane's
//               P V(g - 1) and Q K^T(g + 1); warp 2 also allocates TMEM. One issuing warp per lane:
//               issuing ~12 tcgen05.mma per step from one warp that shares its SM sub-partition with
//               two softmax warps was the bottleneck (profiles/trace_fa_r02.txt)
//   warps 4-7   softmax, lane A (thread = query row); warps 8-11 lane B
//   warps 12-15 epilogue of whichever lane finishes a query block (polls both)
// One step = one 64-key block. TMEM per lane: S0 | S1 (64 columns each) | O (128): S is double
// buffered, so Q K^T(n+1) runs while the softmax works on S(n); P(n) is written as bf16 over
// S(n)'s own columns and Q K^T(n+2) reuses them after P V(n) (tcgen05 executes in issue order).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

namespace fa {
constexpr int BQ = 128, BK = 64, D = 128;
constexpr uint32_t TILE_BYTES = BK * D * 2;  // one key block, 16 KB
constexpr uint32_t PAIR_BYTES = 2 * TILE_BYTES;
constexpr uint32_t Q_BYTES = BQ * D * 2;     // 32 KB
// linsel (persistent): phi(Q) of two tiles, Hc, and a ring of (V_j, phi(K~_j)) stages that runs
// across tiles
constexpr int LS_NST = 4;
constexpr uint32_t LS_OFF_PHIQ = 0, LS_OFF_HC = 2 * Q_BYTES, LS_OFF_RING = LS_OFF_HC + Q_BYTES;
constexpr uint32_t LS_SMEM = LS_OFF_RING + LS_NST * PAIR_BYTES + 1024;  // 225 KB (+ alignment slack)
// attn: Q of both lanes, then per lane a K ring and a V ring of single key blocks
constexpr int NK = 2, NV = 3;
constexpr uint32_t AT_OFF_Q = 0, AT_OFF_K = 2 * Q_BYTES, AT_OFF_V = AT_OFF_K + 2 * NK * TILE_BYTES;
constexpr uint32_t AT_SMEM = AT_OFF_V + 2 * NV * TILE_BYTES + 1024;  // 225 KB (+ alignment slack)
constexpr float RESCALE_LOG2 = 8.0f;
constexpr int AT_THREADS = 512;
}  // namespace fa

__device__ __forceinline__ float fa_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <uint32_t N>
__device__ __forceinline__ void fa_reg_alloc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void fa_reg_dealloc() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

// Bounded waits in analysis builds (-DSLA2_FA_WATCHDOG): a wait that spins ~seconds prints its
// site and traps instead of hanging the GPU.
#ifdef SLA2_FA_WATCHDOG
__device__ __forceinline__ void fa_wait_wd(uint64_t* bar, uint32_t parity, int site) {
    for (long long it = 0; !mbar_try_wait(bar, parity); ++it) {
        if (it == (1ll << 25)) {
            printf("sla2 sparse_fa HANG block %d warp %d lane %d line %d parity %u\n", blockIdx.x, threadIdx.x >> 5,
                   threadIdx.x & 31, site, parity);
            __trap();
        }
    }
}
#define FA_WAIT(bar, par) fa_wait_wd(bar, par, __LINE__)
#else
#define FA_WAIT(bar, par) mbar_wait(bar, par)
#endif

__device__ __forceinline__ uint8_t* fa_align1k(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ================================================================================ linsel
struct LinSelParams {
    const int32_t* kv_idx;
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* ztot;  // [BH][D]
    const float* zblk;  // [BH][tn][D]
    const float* htot;  // [BH][D][D] fp32
    __nv_bfloat16* ol;  // [BH][N][D]
    int N, tm, tn, ntiles;
};

// This CTA's next query block (tile id >= t, in steps of gridDim.x) whose row keeps fewer than
// tn key blocks (rows that keep every block have no linear branch), or -1.
__device__ __forceinline__ int ls_next(const LinSelParams& p, int t, int& nb) {
    for (; t < p.ntiles; t += (int)gridDim.x) {
        nb = p.kv_cnt ? p.kv_cnt[t] : p.kappa;
        if (nb < p.tn) return t;
    }
    return -1;
}

__global__ void __launch_bounds__(256, 1)
    sla2_linsel_kernel(const __grid_constant__ CUtensorMap tmPhiQ, const __grid_constant__ CUtensorMap tmPhiK,
                       const __grid_constant__ CUtensorMap tmV, const LinSelParams p) {
    using namespace fa;
    extern __shared__ uint8_t ls_smem_raw[];
    uint8_t* smem = fa_align1k(ls_smem_raw);
    __shared__ uint64_t bar_full[LS_NST], bar_empty[LS_NST], bar_q_full[2], bar_q_free[2], bar_hs_full[2],
        bar_h_free[2], bar_zc_ready[2], bar_zc_free[2], bar_hc_ready, bar_lin_full, bar_lin_free;
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(16) float sZc[2][D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < LS_NST; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_q_full[b], 1);
            mbar_init(&bar_q_free[b], 1);
            mbar_init(&bar_hs_full[b], 1);
            mbar_init(&bar_h_free[b], 4);
            mbar_init(&bar_zc_ready[b], 1);
            mbar_init(&bar_zc_free[b], 4);
        }
        mbar_init(&bar_hc_ready, 4);
        mbar_init(&bar_lin_full, 1);
        mbar_init(&bar_lin_free, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t sbase = smem_u32(smem);
    constexpr uint32_t TM_LIN = 256;  // Hsel buffers at 0 and 128

    if (warp == 0) {
        // ============ TMA: (V_j, phi(K~_j)) of every kept block, one box per lane, across tiles ============
        if (lane == 0) {
            tma_prefetch_desc(&tmV);
            tma_prefetch_desc(&tmPhiK);
        }
        const uint64_t pol = policy_evict_last();
        int g = 0, nb = 0;
        for (int t = ls_next(p, blockIdx.x, nb); t >= 0; t = ls_next(p, t + (int)gridDim.x, nb)) {
            const int bh = t / p.tm;
            const int32_t* idx = p.kv_idx + (int64_t)t * p.kstride;
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % LS_NST;
                if (lane == 0) {
                    if (g >= LS_NST) FA_WAIT(&bar_empty[s], (uint32_t)(((g / LS_NST) - 1) & 1));
                    mbar_arrive_expect_tx(&bar_full[s], PAIR_BYTES);
                }
                __syncwarp();
                if (lane < 4)  // lanes 0-1: V halves, 2-3: phi(K~) halves
                    tma_load_3d_hint(smem + LS_OFF_RING + s * PAIR_BYTES + lane * 8192, lane < 2 ? &tmV : &tmPhiK,
                                     (lane & 1) * 64, idx[j] * BK, bh, &bar_full[s], pol);
            }
        }
    } else if (warp == 1) {
        // ============ MMA: Hsel(k) = sum_sel phi(K~_j)^T V_j into buffer k & 1 (A = phi^T, B = V,
        // both MN-major); lin(k - 1) = phi(Q) Hc as soon as the epilogue has built Hc(k - 1) ============
        constexpr uint32_t ID_HS = idesc_bf16(128, 128, true, true);
        constexpr uint32_t ID_LIN = idesc_bf16(128, 128, false, true);
        const uint32_t tm = warp_uniform(tmem);
        const uint32_t sb = warp_uniform(sbase);
        int g = 0, k = 0, nb = 0;
        bool lin_pending = false;
        auto issue_lin = [&](int kk) {  // tile kk's phi(Q) Hc
            FA_WAIT(&bar_hc_ready, (uint32_t)(kk & 1));
            FA_WAIT(&bar_q_full[kk & 1], (uint32_t)((kk >> 1) & 1));
            if (kk >= 1) FA_WAIT(&bar_lin_free, (uint32_t)((kk - 1) & 1));
            tc_fence_after();
            const uint64_t dA = sdesc_sw128(sb + LS_OFF_PHIQ + (kk & 1) * Q_BYTES, 16, 1024);
            const uint64_t dB = sdesc_sw128(sb + LS_OFF_HC, 16384, 1024);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                umma_bf16_ss_w(tm + TM_LIN, dA + (((ks >> 2) * 16384 + (ks & 3) * 32) >> 4), dB + ((ks * 2048) >> 4),
                               ID_LIN, ks > 0);
            umma_commit_w(&bar_lin_full);
            umma_commit_w(&bar_q_free[kk & 1]);
        };
        for (int t = ls_next(p, blockIdx.x, nb); t >= 0; t = ls_next(p, t + (int)gridDim.x, nb), ++k) {
            const uint32_t tH = tm + (uint32_t)(k & 1) * 128;
            if (k >= 2) {
                FA_WAIT(&bar_h_free[k & 1], (uint32_t)(((k >> 1) - 1) & 1));  // the epilogue read Hsel(k - 2)
                tc_fence_after();
            }
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % LS_NST;
                FA_WAIT(&bar_full[s], (uint32_t)((g / LS_NST) & 1));
                tc_fence_after();
                const uint64_t dV = sdesc_sw128(sb + LS_OFF_RING + s * PAIR_BYTES, 8192, 1024);
                const uint64_t dP = dV + (TILE_BYTES >> 4);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    umma_bf16_ss_w(tH, dP + ((ks * 2048) >> 4), dV + ((ks * 2048) >> 4), ID_HS, (j > 0 || ks > 0));
                umma_commit_w(&bar_empty[s]);
                if (lin_pending && mbar_test_wait(&bar_hc_ready, (uint32_t)((k - 1) & 1))) {
                    issue_lin(k - 1);
                    lin_pending = false;
                }
            }
            umma_commit_w(&bar_hs_full[k & 1]);
            if (lin_pending) issue_lin(k - 1);
            lin_pending = true;
        }
        if (lin_pending) issue_lin(k - 1);
    } else if (warp == 2) {
        // ============ TMA: phi(Q) of tile k into buffer k & 1 once lin(k - 2) has read it ============
        if (lane == 0) tma_prefetch_desc(&tmPhiQ);
        int k = 0, nb = 0;
        for (int t = ls_next(p, blockIdx.x, nb); t >= 0; t = ls_next(p, t + (int)gridDim.x, nb), ++k) {
            const int bh = t / p.tm, i = t - bh * p.tm;
            if (lane == 0) {
                if (k >= 2) FA_WAIT(&bar_q_free[k & 1], (uint32_t)(((k >> 1) - 1) & 1));
                mbar_arrive_expect_tx(&bar_q_full[k & 1], Q_BYTES);
            }
            __syncwarp();
            if (lane < 4)
                tma_load_3d(smem + LS_OFF_PHIQ + (k & 1) * Q_BYTES + lane * 8192, &tmPhiQ, (lane >> 1) * 64,
                            i * BQ + (lane & 1) * 64, bh, &bar_q_full[k & 1]);
        }
    } else if (warp == 3) {
        // ============ Zc = Ztot - sum_sel z_j per tile (lane: 4 features) ============
        int k = 0, nb = 0;
        for (int t = ls_next(p, blockIdx.x, nb); t >= 0; t = ls_next(p, t + (int)gridDim.x, nb), ++k) {
            const int bh = t / p.tm;
            const int32_t* idx = p.kv_idx + (int64_t)t * p.kstride;
            if (k >= 2) FA_WAIT(&bar_zc_free[k & 1], (uint32_t)(((k >> 1) - 1) & 1));
            const float* zb = p.zblk + (int64_t)bh * p.tn * D + lane * 4;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j0 = 0; j0 < nb; j0 += 8) {
                float4 z[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    z[u] = j0 + u < nb ? *reinterpret_cast<const float4*>(zb + (int64_t)idx[j0 + u] * D)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc.x += z[u].x;
                    acc.y += z[u].y;
                    acc.z += z[u].z;
                    acc.w += z[u].w;
                }
            }
            const float4 zt = *reinterpret_cast<const float4*>(p.ztot + (int64_t)bh * D + lane * 4);
            *reinterpret_cast<float4*>(&sZc[k & 1][lane * 4]) =
                make_float4(zt.x - acc.x, zt.y - acc.y, zt.z - acc.z, zt.w - acc.w);
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_zc_ready[k & 1]);
        }
    } else {
        // ============ epilogue (thread r = TMEM lane r): den, Hc = Htot - Hsel, O_l = lin / den ============
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int k = 0, nb = 0;
        for (int t = ls_next(p, blockIdx.x, nb); t >= 0; t = ls_next(p, t + (int)gridDim.x, nb), ++k) {
            const int bh = t / p.tm, i = t - bh * p.tm;
            // den_r = phi(Q)_r . Zc over the bf16 phi(Q) the MMA uses (K-major SW128 tile)
            FA_WAIT(&bar_q_full[k & 1], (uint32_t)((k >> 1) & 1));
            FA_WAIT(&bar_zc_ready[k & 1], (uint32_t)((k >> 1) & 1));
            float den;
            {
                float2 d2 = make_float2(0.f, 0.f);
                const uint32_t qb = sbase + LS_OFF_PHIQ + (k & 1) * Q_BYTES;
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {
                    const int c = ch * 8;
                    uint32_t w[4];
                    ld_shared_v4(qb + (c >> 6) * 16384 + sw128_off(r, c & 63), w[0], w[1], w[2], w[3]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
                        d2 = __ffma2_rn(f2, *reinterpret_cast<const float2*>(&sZc[k & 1][c + 2 * e]), d2);
                    }
                }
                den = d2.x + d2.y;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_zc_free[k & 1]);
            // Hc = Htot - Hsel, row f = r, as the MN-major B tile [c half 2][f 128][64 c] (bf16). The
            // previous tile's lin MMA (the only reader of Hc) completed before its O_l was read below.
            FA_WAIT(&bar_hs_full[k & 1], (uint32_t)((k >> 1) & 1));
            tc_fence_after();
            const uint32_t hb = sbase + LS_OFF_HC;
            const float4* ht = reinterpret_cast<const float4*>(p.htot + ((int64_t)bh * D + r) * D);
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                float4 hv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) hv[u] = ht[c0 / 4 + u];
                uint32_t hs[32];
                tmem_ld32(tmem + lane_base + (uint32_t)(k & 1) * 128 + c0, hs);
                tmem_ld_wait();
                const float* hf = reinterpret_cast<const float*>(hv);
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const int c = c0 + ch * 8;
                    uint32_t o4[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        o4[e] = pack_bf16(hf[ch * 8 + 2 * e] - __uint_as_float(hs[ch * 8 + 2 * e]),
                                          hf[ch * 8 + 2 * e + 1] - __uint_as_float(hs[ch * 8 + 2 * e + 1]));
                    st_shared_v4(hb + (c >> 6) * 16384 + sw128_off(r, c & 63), o4[0], o4[1], o4[2], o4[3]);
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();  // Hc is read by the tensor core
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bar_h_free[k & 1]);  // Hsel(k) is read: Hsel(k + 2) may overwrite it
                mbar_arrive(&bar_hc_ready);
            }
            // O_l row r = lin_r / den_r (bf16), rows past N dropped
            FA_WAIT(&bar_lin_full, (uint32_t)(k & 1));
            __syncwarp();
            tc_fence_after();
            const bool live = i * BQ + r < p.N;
            const float inv = den > 0.0f ? 1.0f / den : 0.0f;
            uint4* orow = reinterpret_cast<uint4*>(p.ol + ((int64_t)bh * p.N + (int64_t)i * BQ + r) * D);
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tmem + lane_base + TM_LIN + c0, o);
                tmem_ld_wait();
                if (live) {
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch)
                        orow[c0 / 8 + ch] = make_uint4(
                            pack_bf16(__uint_as_float(o[ch * 8 + 0]) * inv, __uint_as_float(o[ch * 8 + 1]) * inv),
                            pack_bf16(__uint_as_float(o[ch * 8 + 2]) * inv, __uint_as_float(o[ch * 8 + 3]) * inv),
                            pack_bf16(__uint_as_float(o[ch * 8 + 4]) * inv, __uint_as_float(o[ch * 8 + 5]) * inv),
                            pack_bf16(__uint_as_float(o[ch * 8 + 6]) * inv, __uint_as_float(o[ch * 8 + 7]) * inv));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_lin_free);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

// ================================================================================ attn
struct AttnParams {
    const int32_t* kv_idx;  // null in dense mode (block j = j)
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* rho;         // [H][tm]
    const __nv_bfloat16* ol;  // [BH][N][D] linear-branch output (sparse mode)
    __nv_bfloat16* out;       // [BH][N][D]
    int N, H, tm, tn, ntiles;
    int last_valid;  // keys in the last (possibly partial) key block
    int dense;
    int pair_kv;  // dense mode, tm even: the lanes take query blocks 2u and 2u + 1 of one head and
                  // share one K / V ring (same key blocks, half the L2 traffic, twice the depth)
    float scale_log2;
#ifdef SLA2_TRACE
    unsigned long long* trace;  // [grid][2 lanes][32 steps][16 events] %globaltimer (analysis build)
#endif
};

#ifdef SLA2_TRACE
__device__ __forceinline__ unsigned long long fa_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define FA_TR(x, g, e) \
    if ((g) < 32) p.trace[(((size_t)blockIdx.x * 2 + (x)) * 32 + (g)) * 16 + (e)] = fa_gtimer()
#else
#define FA_TR(x, g, e)
#endif

struct FaTile {
    int bh, i, nb;
    bool linear;
    const int32_t* idx;  // null: block j = j
};
__device__ __forceinline__ FaTile fa_tile(const AttnParams& p, int t) {
    FaTile r;
    r.bh = t / p.tm;
    r.i = t - r.bh * p.tm;
    if (p.dense) {
        r.nb = p.tn;
        r.idx = nullptr;
        r.linear = false;
    } else {
        r.nb = p.kv_cnt ? p.kv_cnt[(int64_t)r.bh * p.tm + r.i] : p.kappa;
        r.idx = p.kv_idx + ((int64_t)r.bh * p.tm + r.i) * p.kstride;
        r.linear = r.nb != p.tn;
    }
    return r;
}
__device__ __forceinline__ int fa_block(const FaTile& T, int j) { return T.idx ? T.idx[j] : j; }
// lane X's k-th query block of this CTA (or -1)
__device__ __forceinline__ int fa_lane_tile(const AttnParams& p, int x, int k) {
    const int t = p.pair_kv ? 2 * (blockIdx.x + k * (int)gridDim.x) + x : blockIdx.x + (2 * k + x) * (int)gridDim.x;
    return t < p.ntiles ? t : -1;
}

// One lane's walk over its key-block steps (query block ordinal k, block j within it).
struct FaCursor {
    int k, j, t;  // t = tile id, -1 when exhausted
    FaTile T;
};
__device__ __forceinline__ void fa_cur_init(FaCursor& c, const AttnParams& p, int x) {
    c.k = 0;
    c.j = 0;
    c.t = fa_lane_tile(p, x, 0);
    if (c.t >= 0) c.T = fa_tile(p, c.t);
}
__device__ __forceinline__ void fa_cur_next(FaCursor& c, const AttnParams& p, int x) {
    if (++c.j == c.T.nb) {
        c.j = 0;
        ++c.k;
        c.t = fa_lane_tile(p, x, c.k);
        if (c.t >= 0) c.T = fa_tile(p, c.t);
    }
}

__global__ void __launch_bounds__(512, 1)
    sla2_attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
    using namespace fa;
    extern __shared__ uint8_t at_smem_raw[];
    uint8_t* smem = fa_align1k(at_smem_raw);
    __shared__ uint64_t bar_q_full[2], bar_q_free[2], bar_k_full[2][NK], bar_k_empty[2][NK], bar_v_full[2][NV],
        bar_v_empty[2][NV], bar_s_full[2][2], bar_p_full[2][2], bar_pv_done[2], bar_o_ready[2], bar_o_free[2],
        bar_l_full[2], bar_l_free[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ float sL[2][BQ];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);

    if (threadIdx.x == 0) {
        for (int x = 0; x < 2; ++x) {
            mbar_init(&bar_q_full[x], 1);
            mbar_init(&bar_q_free[x], 1);
            for (int b = 0; b < 2; ++b) {  // per S buffer: a lane's steps g and g + 1 may overlap
                mbar_init(&bar_s_full[x][b], 1);
                mbar_init(&bar_p_full[x][b], 4);  // one elected lane per softmax warp
            }
            mbar_init(&bar_pv_done[x], 1);
            mbar_init(&bar_o_ready[x], 1);
            mbar_init(&bar_o_free[x], 4);
            mbar_init(&bar_l_full[x], 4);
            mbar_init(&bar_l_free[x], 4);
            for (int s = 0; s < NK; ++s) {
                mbar_init(&bar_k_full[x][s], 1);
                mbar_init(&bar_k_empty[x][s], p.pair_kv ? 2 : 1);  // shared ring: both issuers release
            }
            for (int s = 0; s < NV; ++s) {
                mbar_init(&bar_v_full[x][s], 1);
                mbar_init(&bar_v_empty[x][s], p.pair_kv ? 2 : 1);
            }
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    // registers: 4 x 64 (TMA / MMA) + 8 x 168 (softmax) + 4 x 104 (epilogue) <= 16 x 128
    if (warp < 4) {
        fa_reg_dealloc<64>();
        if (warp == 0 || warp == 3) {
            // ============ TMA producer of one lane: Q per query block, K and V per key block ============
            // Every box is issued by its own thread: bulk-tensor copies issued by one thread
            // complete one after another (tools/mb_tma.cu), from several threads in parallel.
            const int x = warp == 0 ? 0 : 1;
            if (lane == 0) {
                tma_prefetch_desc(&tmQ);
                tma_prefetch_desc(&tmK);
                tma_prefetch_desc(&tmV);
            }
            const uint64_t pol = policy_evict_last();
            uint8_t* dq = smem + AT_OFF_Q + x * Q_BYTES;
            // shared K / V ring (pair_kv): lane A's producer fills both lanes' slots, lane B's loads Q only
            const bool kv = !p.pair_kv || x == 0;
            const int nk = p.pair_kv ? 2 * NK : NK, nv = p.pair_kv ? 2 * NV : NV;
            uint8_t* dk = smem + AT_OFF_K + (p.pair_kv ? 0 : x * NK * TILE_BYTES);
            uint8_t* dv = smem + AT_OFF_V + (p.pair_kv ? 0 : x * NV * TILE_BYTES);
            uint64_t* kfull = p.pair_kv ? &bar_k_full[0][0] : bar_k_full[x];
            uint64_t* kempty = p.pair_kv ? &bar_k_empty[0][0] : bar_k_empty[x];
            uint64_t* vfull = p.pair_kv ? &bar_v_full[0][0] : bar_v_full[x];
            uint64_t* vempty = p.pair_kv ? &bar_v_empty[0][0] : bar_v_empty[x];
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = fa_lane_tile(p, x, k);
                if (t < 0) break;
                const FaTile T = fa_tile(p, t);
                if (lane == 0) {
                    if (k >= 1) FA_WAIT(&bar_q_free[x], (uint32_t)((k - 1) & 1));  // previous block's last Q K^T done
                    mbar_arrive_expect_tx(&bar_q_full[x], Q_BYTES);
                }
                __syncwarp();
                if (lane < 4)
                    tma_load_3d(dq + lane * 8192, &tmQ, (lane >> 1) * 64, T.i * BQ + (lane & 1) * 64, T.bh, &bar_q_full[x]);
                for (int j = 0; j < T.nb && kv; ++j, ++g) {
                    const int krow = fa_block(T, j) * BK;
                    const int sk = g % nk, sv = g % nv;
                    if (lane == 0) {
                        if (g >= nk) FA_WAIT(&kempty[sk], (uint32_t)(((g / nk) - 1) & 1));
                        mbar_arrive_expect_tx(&kfull[sk], TILE_BYTES);
                        if (g >= nv) FA_WAIT(&vempty[sv], (uint32_t)(((g / nv) - 1) & 1));
                        mbar_arrive_expect_tx(&vfull[sv], TILE_BYTES);
                    }
                    __syncwarp();
                    if (lane < 2)
                        tma_load_3d_hint(dk + sk * TILE_BYTES + lane * 8192, &tmK, lane * 64, krow, T.bh, &kfull[sk], pol);
                    else if (lane < 4)
                        tma_load_3d_hint(dv + sv * TILE_BYTES + (lane - 2) * 8192, &tmV, (lane - 2) * 64, krow, T.bh,
                                         &vfull[sv], pol);
                }
            }
        } else if (warp == 1 || warp == 2) {
            // ============ MMA issuer of one lane (warp 1: A, warp 2: B): Q K^T(0), Q K^T(1), then per
            // step P V(g - 1) and Q K^T(g + 1), which reuses the S / P columns P V(g - 1) has just read
            // (tcgen05 ops of one thread execute in order; tcgen05.commit tracks the issuing thread's
            // own ops, and the lanes share no TMEM columns or shared-memory buffers) ============
            constexpr uint32_t ID_QK = idesc_bf16(128, 64, false, false);
            constexpr uint32_t ID_PV = idesc_bf16(128, 128, false, true);
            const int x = warp - 1;
            const uint32_t tl = warp_uniform(tmem) + (uint32_t)x * 256;  // lane x: S0 | S1 | O
            const uint32_t sb = warp_uniform(sbase);
            const uint64_t dQ = sdesc_sw128(sb + AT_OFF_Q + x * Q_BYTES, 16, 1024);
            const int nk = p.pair_kv ? 2 * NK : NK, nv = p.pair_kv ? 2 * NV : NV;
            const uint64_t dK0 = sdesc_sw128(sb + AT_OFF_K + (p.pair_kv ? 0 : x * NK * TILE_BYTES), 16, 1024);
            const uint64_t dV0 = sdesc_sw128(sb + AT_OFF_V + (p.pair_kv ? 0 : x * NV * TILE_BYTES), 8192, 1024);
            uint64_t* kfull = p.pair_kv ? &bar_k_full[0][0] : bar_k_full[x];
            uint64_t* kempty = p.pair_kv ? &bar_k_empty[0][0] : bar_k_empty[x];
            uint64_t* vfull = p.pair_kv ? &bar_v_full[0][0] : bar_v_full[x];
            uint64_t* vempty = p.pair_kv ? &bar_v_empty[0][0] : bar_v_empty[x];
            FaCursor cq, cp;
            fa_cur_init(cq, p, x);
            fa_cur_init(cp, p, x);
            int gq = 0, gp = 0;  // Q K^T / P V issued
            auto issue_qk = [&]() {
                const int g = gq, sk = g % nk;
                if (cq.j == 0) FA_WAIT(&bar_q_full[x], (uint32_t)(cq.k & 1));
                FA_WAIT(&kfull[sk], (uint32_t)((g / nk) & 1));
                tc_fence_after();
                const uint64_t dK = dK0 + (uint64_t)((sk * TILE_BYTES) >> 4);
                const uint32_t tS = tl + (uint32_t)(g & 1) * 64;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_bf16_ss_w(tS, dQ + (((ks >> 2) * 16384 + (ks & 3) * 32) >> 4),
                                   dK + (((ks >> 2) * 8192 + (ks & 3) * 32) >> 4), ID_QK, ks > 0);
                umma_commit_w(&bar_s_full[x][g & 1]);
                if (lane == 0) FA_TR(x, g, 0);
                umma_commit_w(&kempty[sk]);
                if (cq.j == cq.T.nb - 1) umma_commit_w(&bar_q_free[x]);
                ++gq;
                fa_cur_next(cq, p, x);
            };
            auto issue_pv = [&]() {
                const int g = gp, sv = g % nv;
                FA_WAIT(&bar_p_full[x][g & 1], (uint32_t)((g >> 1) & 1));
                if (lane == 0) FA_TR(x, g, 7);
                if (cp.j == 0 && cp.k >= 1) FA_WAIT(&bar_o_free[x], (uint32_t)((cp.k - 1) & 1));
                FA_WAIT(&vfull[sv], (uint32_t)((g / nv) & 1));
                tc_fence_after();
                const uint64_t dV = dV0 + (uint64_t)((sv * TILE_BYTES) >> 4);
                const uint32_t tP = tl + (uint32_t)(g & 1) * 64;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    umma_bf16_ts_w(tl + 128, tP + ks * 8, dV + ((ks * 2048) >> 4), ID_PV, (cp.j > 0 || ks > 0));
                umma_commit_w(&bar_pv_done[x]);
                if (lane == 0) FA_TR(x, g, 1);
                umma_commit_w(&vempty[sv]);
                if (cp.j == cp.T.nb - 1) umma_commit_w(&bar_o_ready[x]);
                ++gp;
                fa_cur_next(cp, p, x);
            };
            for (int u = 0; u < 2 && cq.t >= 0; ++u) issue_qk();
            while (gp < gq) {
                issue_pv();
                if (cq.t >= 0) issue_qk();
            }
        }
    } else if (warp < 12) {
        fa_reg_alloc<168>();
        // ============ softmax of lane x: thread = query row r, one key block per step ============
        const int x = (warp - 4) >> 2;
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tl = tmem + lane_base + (uint32_t)x * 256, tO = tl + 128;
        const float sc = p.scale_log2;
        const float2 sc2 = make_float2(sc, sc);
        int g = 0;  // steps consumed by this lane
        for (int k = 0;; ++k) {
            const int t = fa_lane_tile(p, x, k);
            if (t < 0) break;
            const FaTile T = fa_tile(p, t);
            const int nb = T.nb;
            // ragged N: the partial last key block's padded keys get -inf
            const int jtail = (p.last_valid < BK && fa_block(T, nb - 1) == p.tn - 1) ? nb - 1 : -1;
            float m = -INFINITY, l = 0.0f;
            for (int j = 0; j < nb; ++j, ++g) {
                FA_WAIT(&bar_s_full[x][g & 1], (uint32_t)((g >> 1) & 1));
                __syncwarp();
                tc_fence_after();
                if (r == 0) FA_TR(x, g, 2);
                const uint32_t tS = tl + (uint32_t)(g & 1) * 64;
                uint32_t sr[64];
                tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                tmem_ld_wait();
                if (r == 0) FA_TR(x, g, 8);
                if (j == jtail) {
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
                if (r == 0) FA_TR(x, g, 9);
                if (j == 0) {
                    m = mx;
                } else if (__any_sync(0xffffffffu, mx > m + RESCALE_LOG2)) {
                    // lazy rescale (threshold 2^8): O must hold P V(g-1) first
                    const float mnew = fmaxf(m, mx);
                    const float corr = fa_exp2(m - mnew);
                    FA_WAIT(&bar_pv_done[x], (uint32_t)((g - 1) & 1));
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
                // P = exp2(S scale - m) as bf16 over the block's own first 32 S columns
                const float2 nm2 = make_float2(-m, -m);
                float2 rs = make_float2(0.f, 0.f);
                uint32_t w[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float2 v2 = __ffma2_rn(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])),
                                                 sc2, nm2);
                    const float2 pe = make_float2(fa_exp2(v2.x), fa_exp2(v2.y));
                    rs = __fadd2_rn(rs, pe);
                    w[e] = pack_bf16(pe.x, pe.y);
                }
                if (r == 0) FA_TR(x, g, 10);
                tmem_st32(tS, w);
                l += rs.x + rs.y;
                tmem_st_wait();
                if (r == 0) FA_TR(x, g, 11);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_p_full[x][g & 1]);
                if (lane == 0) FA_TR(x, g, (warp & 3) == 0 ? 3 : 3 + (warp & 3));
            }
            // the block's row sums to the epilogue (sL[x] is free once it read the previous ones)
            if (k >= 1) FA_WAIT(&bar_l_free[x], (uint32_t)((k - 1) & 1));
            sL[x][r] = l;
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_l_full[x]);
        }
    } else {
        fa_reg_dealloc<104>();  // below the launch allocation: .dec
        // ============ epilogue: out = alpha O / l + (1 - alpha) O_l, whichever lane is ready ============
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int ke[2] = {0, 0};
        int te[2] = {fa_lane_tile(p, 0, 0), fa_lane_tile(p, 1, 0)};
        while (te[0] >= 0 || te[1] >= 0) {
            // each warp serves its own 32 rows of every query block once, in its own order
            int x = -1;
            for (int y = 0; y < 2 && x < 0; ++y)
                if (te[y] >= 0 && mbar_try_wait_ns(&bar_o_ready[y], (uint32_t)(ke[y] & 1), 200)) x = y;
            x = __shfl_sync(0xffffffffu, x, 0);
            if (x < 0) continue;
            const FaTile T = fa_tile(p, te[x]);
            const bool live = T.i * BQ + r < p.N;
            const int64_t grow = (int64_t)T.bh * p.N + (int64_t)T.i * BQ + r;
            float alpha = 1.0f;
            const uint4* og = reinterpret_cast<const uint4*>(p.ol + grow * D);
            const bool lin = T.linear && live;
            uint4 olr[4];  // O_l columns of the current 32-column chunk
            if (T.linear) {
                const float xr = p.rho[(int64_t)(T.bh % p.H) * p.tm + T.i];
                const float a = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-xr)));
                alpha = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);  // attention.hpp:17-22
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) olr[u] = lin ? og[u] : make_uint4(0u, 0u, 0u, 0u);
            FA_WAIT(&bar_l_full[x], (uint32_t)(ke[x] & 1));
            const float l = sL[x][r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_l_free[x]);
            tc_fence_after();
            const float a_l = alpha / l, b = 1.0f - alpha;
            const uint32_t tO = tmem + lane_base + (uint32_t)x * 256 + 128;
            uint4* orow = reinterpret_cast<uint4*>(p.out + grow * D);
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tO + c0, o);
                tmem_ld_wait();
                if (c0 == 96) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bar_o_free[x]);  // the lane's next P V(0) may overwrite O
                }
                uint4 cur[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) cur[u] = olr[u];
                if (c0 < 96) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) olr[u] = lin ? og[(c0 + 32) / 8 + u] : make_uint4(0u, 0u, 0u, 0u);
                }
                if (live) {
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t w[4];
                        const uint32_t* lw = reinterpret_cast<const uint32_t*>(&cur[ch]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 lf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&lw[e]));
                            const float v0 = fmaf(b, lf.x, __uint_as_float(o[ch * 8 + 2 * e]) * a_l);
                            const float v1 = fmaf(b, lf.y, __uint_as_float(o[ch * 8 + 2 * e + 1]) * a_l);
                            w[e] = pack_bf16(v0, v1);
                        }
                        orow[c0 / 8 + ch] = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
            }
            ++ke[x];
            te[x] = fa_lane_tile(p, x, ke[x]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

// ================================================================================ launch
bool sparse_fa_eligible(const SparseLaunch& a) {
    return a.bq == 128 && a.bk == 64 && a.d == 128 && a.o_s == nullptr && a.o_l == nullptr && a.big_l == nullptr &&
           a.h_blocks == nullptr && a.z_blocks == nullptr && a.s_first == nullptr &&
           (a.dense || (a.phiq != nullptr && a.tm_phiq != nullptr && a.ol != nullptr));
}

cudaError_t launch_linsel(const SparseLaunch& a, cudaStream_t st, int* launches) {
    LinSelParams lp;
    lp.kv_idx = a.kv_idx;
    lp.kv_cnt = a.kv_cnt;
    lp.kstride = a.kstride;
    lp.kappa = a.kappa;
    lp.ztot = a.ztot;
    lp.zblk = a.zblk;
    lp.htot = a.htot;
    lp.ol = (__nv_bfloat16*)a.ol;
    lp.N = a.N;
    lp.tm = a.tm;
    lp.tn = a.tn;
    lp.ntiles = (int)(a.B * a.H) * a.tm;
    cudaError_t e = ensure_smem_attr((const void*)sla2_linsel_kernel, (int)fa::LS_SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    sla2_linsel_kernel<<<lp.ntiles < sms ? lp.ntiles : sms, 256, fa::LS_SMEM, st>>>(*a.tm_phiq, *a.tm_phik, *a.tm_v,
                                                                                    lp);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sparse_fa(const SparseLaunch& a, cudaStream_t st, int* launches) {
    const int ntiles = (int)(a.B * a.H) * a.tm;
    if (!a.dense) {
        const cudaError_t e = launch_linsel(a, st, launches);
        if (e != cudaSuccess) return e;
    }
    AttnParams p;
    p.kv_idx = a.dense ? nullptr : a.kv_idx;
    p.kv_cnt = a.dense ? nullptr : a.kv_cnt;
    p.kstride = a.kstride;
    p.kappa = a.kappa;
    p.rho = a.rho;
    p.ol = (const __nv_bfloat16*)a.ol;
    p.out = (__nv_bfloat16*)a.out;
    p.N = a.N;
    p.H = (int)a.H;
    p.tm = a.tm;
    p.tn = a.tn;
    p.ntiles = ntiles;
    p.last_valid = a.N - (a.tn - 1) * fa::BK;
    p.dense = a.dense;
    p.pair_kv = a.dense && (a.tm % 2 == 0);
    p.scale_log2 = a.inv_sqrt_d * 1.4426950408889634f;
#ifdef SLA2_TRACE
    extern unsigned long long* g_trace_buf;
    p.trace = g_trace_buf;
#endif
    cudaError_t e = ensure_smem_attr((const void*)sla2_attn_kernel, (int)fa::AT_SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // two query blocks per CTA: enough CTAs that every SM gets its two lanes
    const int grid = (ntiles + 1) / 2 < sms ? (ntiles + 1) / 2 : sms;
    sla2_attn_kernel<<<grid, fa::AT_THREADS, fa::AT_SMEM, st>>>(*a.tm_q, *a.tm_k, *a.tm_v, p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
