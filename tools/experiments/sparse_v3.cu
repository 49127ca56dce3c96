// sparse_v3.cu -- the persistent SLA2 sparse + linear + alpha-blend forward (sm_100a, bf16).
//
// Same algorithm as sparse_bf16.cu (the per-query-block loop of sla2_forward_blockwise,
// attention.hpp:484-558, with block_scores_qk / block_product_pv, 372-415). What bounds a
// key-block pair on B200 shaped this version (tools/mb_tmem.cu, profiles/):
//
//  * the softmax, not the tensor pipe: one softmax warp per SM sub-partition issuing scalar
//    FFMA/FADD beside MUFU.EX2 takes ~1400 cycles per 128 x 128 pass; two warps per
//    sub-partition with packed FFMA2/FADD2 reach the MUFU floor (~1030 cycles, 16 ex2/clk/SM).
//    So 8 softmax warps: warp pair (w, w+4) shares TMEM lanes 32(w%4).. and each takes ONE key
//    block of the pair (64 columns). The row max is exchanged once per tile (shared memory +
//    named barrier); afterwards a `bar.red.or` per pair tells both halves whether either needs
//    the lazy rescale, and only then are the maxima exchanged again;
//  * the single S buffer: QK^T of pair n+1 waited for the softmax to drain S(n). Now S is
//    double-buffered and P(n) is written over S(n)'s own columns (FA4-style aliasing), so the
//    tensor pipe runs QK^T(n+1) and PV(n-1) while the softmax works on n. QK^T(n+2) reuses
//    buffer n&1 after PV(n) in issue order (tcgen05.mma executes in order);
//  * the epilogue: O leaves TMEM right after the tile's last MMA (as packed bf16 alpha/l * O in
//    registers), so the next tile's first PV is not held behind the linear term. The linear
//    numerator phi(Q) (Htot - Hsel) is one SS MMA into the Hsel columns (A = phi(Q), TMA-loaded
//    over the tile's finished Q buffer; B = Hc built by the epilogue in a V-ring slot), and the
//    epilogue blends out = (alpha/l) O + ((1 - alpha)/den) lin (attention.hpp:532-557).
//
// Roles (16 warps, one CTA per SM, tiles (b, h, query block) round robin):
//   warp 0     TMA: Q (two buffers) and the K-pair ring
//   warp 1     MMA issuer (whole warp, elect.sync inside each tcgen05 op)
//   warp 2     TMEM allocator; TMA: the V / phi(K~) ring (+ one slot per tile for Hc)
//   warp 3     Zc = Ztot - sum_sel z_j (the linear denominators); TMA: phi(Q) after the tile's
//              last Q K^T
//   warps 4-11 softmax (half h = block 2n+h of pair n, thread = query row)
//   warps 12-15 epilogue of the previous tile (thread = query row)
// TMEM (512 columns): S/P buffer 0 | S/P buffer 1 | O | Hsel, then the tile's linear product.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

namespace v3 {
constexpr int BQ = 128, BK = 64, D = 128;
constexpr int NKP = 2, NSV = 3;                // K pair ring, V / phi(K~) ring (one slot per tile holds Hc)
constexpr uint32_t Q_BYTES = BQ * D * 2;       // 32 KB
constexpr uint32_t TILE_BYTES = BK * D * 2;    // 16 KB
constexpr uint32_t KP_BYTES = 2 * TILE_BYTES;  // a K pair
constexpr uint32_t VS_BYTES = 2 * TILE_BYTES;  // V + phi(K~), or Hc (bf16 128 x 128)
constexpr uint32_t OFF_Q = 0;                  // 2 Q buffers
constexpr uint32_t OFF_K = OFF_Q + 2 * Q_BYTES;
constexpr uint32_t OFF_V = OFF_K + NKP * KP_BYTES;
constexpr uint32_t SMEM_BYTES = OFF_V + NSV * VS_BYTES;  // 224 KB (+ < 3 KB static: the 227 KB limit)
constexpr uint32_t TM_SP0 = 0, TM_O = 256, TM_H = 384;   // S/P buffer b at b * 128
constexpr float RESCALE_LOG2 = 8.0f;
constexpr int NTHREADS = 512;
}  // namespace v3

struct SparseV3Params {
    const int32_t* kv_idx;
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* rho;
    const float* ztot;
    const float* zblk;
    const __nv_bfloat16* htot16;  // [BH][D][D] bf16 (the epilogue forms Hc = Htot - Hsel from it)
    const __nv_bfloat16* phiq;    // [BH][N][D] bf16 phi(Q) rows (router front)
    __nv_bfloat16* out;           // [BH][N][D]
    int N, H, tm, tn, ntiles;
    int last_valid;
    float scale_log2;
#ifdef SLA2_TRACE
    unsigned long long* trace;  // [grid][8 tiles][32 events] %globaltimer stamps (analysis build)
#endif
};

__device__ __forceinline__ float v3_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <uint32_t N>
__device__ __forceinline__ void v3_reg_alloc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void v3_reg_dealloc() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
// OR of pred over the nthreads threads of named barrier id (the two softmax warps of a lane quarter)
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t nthreads, bool pred) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %3, 0;\n\t"
        "bar.red.or.pred q, %1, %2, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(id), "r"(nthreads), "r"(pred ? 1u : 0u)
        : "memory");
    return r != 0;
}

#ifdef SLA2_TRACE
__device__ __forceinline__ unsigned long long v3_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define V3_TR(k, e) \
    if ((k) < 8) p.trace[((size_t)blockIdx.x * 8 + (k)) * 96 + (e)] = v3_gtimer()
#else
#define V3_TR(k, e)
#endif

#ifdef SLA2_V2_WATCHDOG
__device__ __forceinline__ void v3_wait(uint64_t* bar, uint32_t parity, int site) {
    for (long long it = 0; !mbar_try_wait(bar, parity); ++it) {
        if (it == (1ll << 26)) {
            printf("sla2_sparse_v3 HANG block %d warp %d lane %d line %d parity %u\n", blockIdx.x, threadIdx.x >> 5,
                   threadIdx.x & 31, site, parity);
            __trap();
        }
    }
}
#define V3_WAIT(bar, par) v3_wait(bar, par, __LINE__)
#else
#define V3_WAIT(bar, par) mbar_wait(bar, par)
#endif

// Everything about tile t every role needs (all roles walk the same tile sequence).
struct V3Tile {
    int64_t bh;
    int i, nb, npair;
    bool linear;
    const int32_t* idx;
};
__device__ __forceinline__ V3Tile v3_tile(const SparseV3Params& p, int t) {
    V3Tile r;
    r.bh = t / p.tm;
    r.i = t - (int)r.bh * p.tm;
    r.nb = p.kv_cnt ? p.kv_cnt[r.bh * p.tm + r.i] : p.kappa;
    r.npair = (r.nb + 1) >> 1;
    r.linear = r.nb != p.tn;
    r.idx = p.kv_idx + (r.bh * p.tm + r.i) * (int64_t)p.kstride;
    return r;
}

// S(pair gg) = Q [K_2n; K_2n+1]^T into S/P buffer gg & 1 (whole warp issues)
__device__ __forceinline__ void v3_issue_qk(uint64_t* k_full, uint64_t* k_empty, uint64_t* s_full, int gg,
                                            uint32_t sbase, uint32_t tm, int pb, bool two) {
    using namespace v3;
    const int s = gg % NKP;
    V3_WAIT(&k_full[s], (uint32_t)((gg / NKP) & 1));
    tc_fence_after();
    const uint32_t idq = two ? idesc_bf16(128, 128, false, false) : idesc_bf16(128, 64, false, false);
    const uint64_t dQ = sdesc_sw128(sbase + OFF_Q + pb * Q_BYTES, 16, 1024);
    const uint64_t dK = sdesc_sw128(sbase + OFF_K + s * KP_BYTES, 16, 1024);
    const uint32_t dS = tm + TM_SP0 + (uint32_t)(gg & 1) * 128;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
        umma_bf16_ss_w(dS, dQ + off, dK + off, idq, ks > 0);
    }
    umma_commit_w(&s_full[gg & 1]);
    umma_commit_w(&k_empty[s]);
}
// lin = phi(Q) Hc of tile kk into the Hsel columns: A = phi(Q) (K-major, TMA-loaded over the
// tile's Q buffer), B = Hc (MN-major) in the tile's Hc slot. Frees the Hc slot when done.
__device__ __forceinline__ void v3_lin_mma(uint64_t* lin_ready, uint64_t* phiq_full, uint64_t* lin_done,
                                           uint64_t* hc_empty, int kk, bool linear, uint32_t sbase, uint32_t tm,
                                           int hc) {
    using namespace v3;
    V3_WAIT(lin_ready, (uint32_t)(kk & 1));
    V3_WAIT(&phiq_full[kk & 1], (uint32_t)((kk >> 1) & 1));
    tc_fence_after();
    if (linear) {
        const uint64_t dA = sdesc_sw128(sbase + OFF_Q + (kk & 1) * Q_BYTES, 16, 1024);
        const uint64_t dB = sdesc_sw128(sbase + OFF_V + hc * VS_BYTES, 16384, 1024);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t offa = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
            umma_bf16_ss_w(tm + TM_H, dA + offa, dB + ((ks * 2048) >> 4), idesc_bf16(128, 128, false, true), ks > 0);
        }
    }
    umma_commit_w(lin_done);
    umma_commit_w(hc_empty);
}

__global__ void __launch_bounds__(512, 1)
    sla2_sparse_v3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmPhi,
                          const __grid_constant__ CUtensorMap tmPhiQ, const SparseV3Params p) {
    using namespace v3;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    __shared__ uint64_t bar_q_full[2], bar_qk_done[2], bar_phiq_full[2], bar_k_full[NKP], bar_k_empty[NKP],
        bar_v_full[NSV], bar_v_empty[NSV], bar_s_full[2], bar_p_full[2], bar_pv_done[2], bar_tile_done, bar_sm_done,
        bar_l_free, bar_o_free, bar_lin_ready, bar_lin_done, bar_hl_free, bar_zc_ready, bar_zc_free;
    __shared__ uint32_t tmem_base_sh;
    __shared__ float sZc[D];        // the tile's Zc (single buffer: zc_ready / zc_free)
    __shared__ float sXch[2][BQ];   // row-max exchange between the two softmax halves
    __shared__ float sLp[2][BQ];    // per-half row sums l of the tile (single buffer: sm_done / l_free)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = p.ntiles, G = gridDim.x;
    auto sQ = [&](int b) { return smem + OFF_Q + b * Q_BYTES; };
    auto sKp = [&](int s) { return smem + OFF_K + s * KP_BYTES; };
    auto sV = [&](int s) { return smem + OFF_V + s * VS_BYTES; };

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();  // SW128 tiles need 1 KB alignment
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_q_full[b], 1);
            mbar_init(&bar_qk_done[b], 1);
            mbar_init(&bar_phiq_full[b], 1);
            mbar_init(&bar_s_full[b], 1);
            mbar_init(&bar_p_full[b], 8);  // one elected lane per softmax warp
            mbar_init(&bar_pv_done[b], 1);
        }
        for (int s = 0; s < NKP; ++s) {
            mbar_init(&bar_k_full[s], 1);
            mbar_init(&bar_k_empty[s], 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(&bar_v_full[s], 1);
            mbar_init(&bar_v_empty[s], 1);
        }
        mbar_init(&bar_tile_done, 1);
        mbar_init(&bar_sm_done, 256);
        mbar_init(&bar_l_free, 128);
        mbar_init(&bar_o_free, 128);
        mbar_init(&bar_lin_ready, 128);
        mbar_init(&bar_lin_done, 1);
        mbar_init(&bar_hl_free, 128);
        mbar_init(&bar_zc_ready, 1);
        mbar_init(&bar_zc_free, 128);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    // registers per thread: 80 (warps 0-3) + 2 x 128 (softmax) + 176 (epilogue) = 512 = 4 x 128,
    // the launch allocation
    if (warp < 4) {
        v3_reg_dealloc<80>();
        if (warp == 0) {
            // ============ TMA: Q (two buffers) and the K-pair ring ============
            // Each box is issued by its own lane: TMA instructions from one thread complete one
            // after another (~600 cycles per 8 KB box, tools/mb_tma.cu), from several lanes in parallel.
            if (lane == 0) {
                tma_prefetch_desc(&tmQ);
                tma_prefetch_desc(&tmK);
            }
            const uint64_t pol = policy_evict_last();
            auto load_q = [&](uint64_t* bar, uint8_t* dst, int qrow, int hz) {
                if (lane == 0) mbar_arrive_expect_tx(bar, Q_BYTES);
                __syncwarp();
                if (lane < 4)
                    tma_load_3d(dst + lane * 8192, &tmQ, (lane >> 1) * 64, qrow + (lane & 1) * 64, hz, bar);
            };
            int64_t gk = 0;
            int t = blockIdx.x;
            if (t < nt) {
                const V3Tile T0 = v3_tile(p, t);
                load_q(&bar_q_full[0], sQ(0), T0.i * BQ, (int)T0.bh);
            }
            for (int k = 0; t < nt; ++k, t += G) {
                const V3Tile T = v3_tile(p, t);
                for (int n = 0; n < T.npair; ++n, ++gk) {
                    const int s = (int)(gk % NKP);
                    const int cnt = min(2, T.nb - 2 * n);
                    if (lane == 0) {
                        if (gk >= NKP) V3_WAIT(&bar_k_empty[s], (uint32_t)(((gk / NKP) - 1) & 1));
                        if (n < 8) V3_TR(k, 64 + n);
                        mbar_arrive_expect_tx(&bar_k_full[s], cnt * TILE_BYTES);
                    }
                    __syncwarp();
                    if (lane < 2 * cnt) {  // lane = (block b, 64-column half c)
                        const int b = lane >> 1, c = lane & 1;
                        const int krow = T.idx[2 * n + b] * BK;
                        tma_load_3d_hint(sKp(s) + c * 16384 + b * 8192, &tmK, c * 64, krow, (int)T.bh, &bar_k_full[s],
                                         pol);
                    }
                }
                // Q of tile k+1 into buffer (k+1)&1, which held phi(Q) of tile k-1 until its lin MMA
                if (t + G < nt) {
                    const V3Tile T1 = v3_tile(p, t + G);
                    if (lane == 0 && k >= 1) V3_WAIT(&bar_lin_done, (uint32_t)((k - 1) & 1));
                    load_q(&bar_q_full[(k + 1) & 1], sQ((k + 1) & 1), T1.i * BQ, (int)T1.bh);
                }
            }
        } else if (warp == 2) {
            // ============ TMA: the V / phi(K~) ring; one slot per tile for the epilogue's Hc ============
            if (lane == 0) {
                tma_prefetch_desc(&tmV);
                tma_prefetch_desc(&tmPhi);
            }
            const uint64_t pol = policy_evict_last();
            int64_t gv = 0;
            for (int t = blockIdx.x; t < nt; t += G) {
                const V3Tile T = v3_tile(p, t);
#ifdef SLA2_ABL_NOHSEL
                const bool ldphi = false;
#else
                const bool ldphi = T.linear;
#endif
                for (int j = 0; j <= T.nb; ++j, ++gv) {
                    const int s = (int)(gv % NSV);
                    if (lane == 0) {
                        if (gv >= NSV) V3_WAIT(&bar_v_empty[s], (uint32_t)(((gv / NSV) - 1) & 1));
                        if (j == T.nb)  // the Hc slot: allocated, not loaded
                            mbar_arrive(&bar_v_full[s]);
                        else
                            mbar_arrive_expect_tx(&bar_v_full[s], ldphi ? 2 * TILE_BYTES : TILE_BYTES);
                    }
                    __syncwarp();
                    if (j < T.nb && lane < (ldphi ? 4 : 2)) {  // lane = (tensor V / phi, 64-column half)
                        const int krow = T.idx[j] * BK, hz = (int)T.bh, c = lane & 1;
                        const CUtensorMap* m = lane < 2 ? &tmV : &tmPhi;
                        tma_load_3d_hint(sV(s) + (lane >> 1) * TILE_BYTES + c * 8192, m, c * 64, krow, hz, &bar_v_full[s],
                                         pol);
                    }
                }
            }
        } else if (warp == 1) {
            // ============ MMA issuer ============
            constexpr uint32_t ID_PV = idesc_bf16(128, 128, false, true);
            constexpr uint32_t ID_HS = idesc_bf16(128, 128, true, true);
            const uint32_t tm = warp_uniform(tmem);
            const uint32_t sbase = warp_uniform(smem_u32(smem));
            const uint64_t dVm = sdesc_sw128(sbase + OFF_V, 8192, 1024);
            int g = 0, gv = 0;  // global pair / V-slot counters
            int k = 0;
            bool prev_linear = false;
            int prev_hc = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V3Tile T = v3_tile(p, t);
                const int nbu = (int)warp_uniform((uint32_t)T.nb);
                const int npu = (nbu + 1) >> 1;
                const bool lin = T.linear;
                const int pb = k & 1;
                V3_WAIT(&bar_q_full[pb], (uint32_t)((k >> 1) & 1));
                tc_fence_after();
                if (lane == 0) V3_TR(k, 0);
                v3_issue_qk(bar_k_full, bar_k_empty, bar_s_full, g, sbase, tm, pb, nbu > 1);
                if (npu > 1) v3_issue_qk(bar_k_full, bar_k_empty, bar_s_full, g + 1, sbase, tm, pb, nbu > 3);
                if (npu <= 2) umma_commit_w(&bar_qk_done[pb]);  // the tile's last Q K^T is issued
                for (int n = 0; n < npu; ++n) {
                    const int gg = g + n;
                    V3_WAIT(&bar_p_full[gg & 1], (uint32_t)((gg >> 1) & 1));
                    tc_fence_after();
                    if (lane == 0 && n < 8) V3_TR(k, 32 + n);
                    if (n == 0 && k > 0) {
                        V3_WAIT(&bar_o_free, (uint32_t)((k - 1) & 1));  // tile k-1's O left TMEM
                        tc_fence_after();
                    }
                    if (lane == 0 && (n < 2 || n == npu - 1)) V3_TR(k, 25 + (n < 2 ? n : 2));
                    if (lane == 0 && n < 8) V3_TR(k, 80 + n);
                    const int j0 = 2 * n, j1 = min(nbu, j0 + 2);
                    const uint32_t aS = tm + TM_SP0 + (uint32_t)(gg & 1) * 128;
                    for (int j = j0; j < j1; ++j) {
                        const int v = gv + j;
                        const int sv = v % NSV;
                        V3_WAIT(&bar_v_full[sv], (uint32_t)((v / NSV) & 1));
                        tc_fence_after();
                        const uint64_t dV = dVm + ((sv * VS_BYTES) >> 4);
                        const uint32_t aP = aS + (uint32_t)(j & 1) * 64;
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            umma_bf16_ts_w(tm + TM_O, aP + ks * 8, dV + ((ks * 2048) >> 4), ID_PV, (j > 0 || ks > 0));
                    }
                    umma_commit_w(&bar_pv_done[gg & 1]);
                    if (lane == 0 && n < 8) V3_TR(k, 40 + n);
                    if (n + 2 < npu) {  // S(n+2) into the buffer PV(n) just read (in-order tensor pipe)
                        if (lane == 0 && n < 8) V3_TR(k, 88 + n);
                        v3_issue_qk(bar_k_full, bar_k_empty, bar_s_full, gg + 2, sbase, tm, pb, 2 * (n + 2) + 1 < nbu);
                        if (lane == 0 && n < 8) V3_TR(k, 48 + n);
                        if (n + 3 == npu) umma_commit_w(&bar_qk_done[pb]);
                    }
                    if (n == 0 && k > 0) {
                        // tile k-1's linear product, then its read-out before this tile's Hsel
                        v3_lin_mma(&bar_lin_ready, bar_phiq_full, &bar_lin_done, &bar_v_empty[prev_hc], k - 1,
                                   prev_linear, sbase, tm, prev_hc);
                        if (lane == 0) V3_TR(k, 22);
                        V3_WAIT(&bar_hl_free, (uint32_t)((k - 1) & 1));
                        tc_fence_after();
                        if (lane == 0) V3_TR(k, 23);
                    }
                    for (int j = j0; j < j1; ++j) {
                        const int sv = (gv + j) % NSV;
#ifdef SLA2_ABL_NOHSEL
                        if (false) {
#else
                        if (lin) {
#endif
                            const uint64_t dV = dVm + ((sv * VS_BYTES) >> 4);
                            const uint64_t dP = dV + (TILE_BYTES >> 4);
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                umma_bf16_ss_w(tm + TM_H, dP + ((ks * 2048) >> 4), dV + ((ks * 2048) >> 4), ID_HS,
                                               (j > 0 || ks > 0));
                        }
                        umma_commit_w(&bar_v_empty[sv]);
                    }
                    if (lane == 0 && n < 8) V3_TR(k, 56 + n);
                }
                umma_commit_w(&bar_tile_done);
                if (lane == 0) V3_TR(k, 24);
                g += npu;
                gv += nbu;
                prev_hc = gv % NSV;  // the tile's Hc slot
                gv += 1;
                prev_linear = lin;
            }
            if (k > 0)
                v3_lin_mma(&bar_lin_ready, bar_phiq_full, &bar_lin_done, &bar_v_empty[prev_hc], k - 1, prev_linear,
                           sbase, tm, prev_hc);
        } else if (warp == 3) {
            // ============ Zc per tile; phi(Q) over the tile's Q after its last Q K^T ============
            if (lane == 0) tma_prefetch_desc(&tmPhiQ);
            int k = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V3Tile T = v3_tile(p, t);
                const int pb = k & 1;
                if (k >= 1) V3_WAIT(&bar_zc_free, (uint32_t)((k - 1) & 1));
                if (T.linear) {
                    const float* zb = p.zblk + T.bh * (int64_t)p.tn * D + lane * 4;
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int j0 = 0; j0 < T.nb; j0 += 32) {
                        const int myj = (j0 + lane < T.nb) ? T.idx[j0 + lane] : 0;
                        const int cnt = min(32, T.nb - j0);
                        for (int u0 = 0; u0 < cnt; u0 += 8) {  // 8 rows in flight per lane
                            float4 z[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const int jj = __shfl_sync(0xffffffffu, myj, (u0 + u) & 31);
                                z[u] = u0 + u < cnt ? *reinterpret_cast<const float4*>(zb + (int64_t)jj * D)
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                acc.x += z[u].x;
                                acc.y += z[u].y;
                                acc.z += z[u].z;
                                acc.w += z[u].w;
                            }
                        }
                    }
                    const float4 zt = *reinterpret_cast<const float4*>(p.ztot + T.bh * D + lane * 4);
                    *reinterpret_cast<float4*>(&sZc[lane * 4]) =
                        make_float4(zt.x - acc.x, zt.y - acc.y, zt.z - acc.z, zt.w - acc.w);
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&bar_zc_ready);
                    V3_WAIT(&bar_qk_done[pb], (uint32_t)((k >> 1) & 1));  // the tile's Q is no longer read
                    if (T.linear)
                        mbar_arrive_expect_tx(&bar_phiq_full[pb], Q_BYTES);
                    else
                        mbar_arrive(&bar_phiq_full[pb]);
                }
                __syncwarp();
                if (T.linear && lane < 4)
                    tma_load_3d(sQ(pb) + lane * 8192, &tmPhiQ, (lane >> 1) * 64, T.i * BQ + (lane & 1) * 64, (int)T.bh,
                                &bar_phiq_full[pb]);
                __syncwarp();
            }
        }
    } else if (warp < 12) {
        // ============ softmax: half h takes block 2n+h of pair n; thread = query row r ============
        const int q4 = warp & 3, h = (warp - 4) >> 2;
        const int r = q4 * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
        const uint32_t bar_x = 1 + q4, bar_r = 5 + q4;  // named barriers of this lane quarter (64 threads)
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        int g = 0, k = 0;
        for (int t = blockIdx.x; t < nt; t += G, ++k) {
            const V3Tile T = v3_tile(p, t);
            const int nb = T.nb, npair = T.npair;
            const bool tail_kept = p.last_valid < BK && T.idx[nb - 1] == p.tn - 1;
            float m = -INFINITY, l = 0.0f;
            for (int n = 0; n < npair; ++n) {
                const int gg = g + n;
                const int b = gg & 1;
                const int j = 2 * n + h;
                const bool has = j < nb;
                V3_WAIT(&bar_s_full[b], (uint32_t)((gg >> 1) & 1));
                __syncwarp();
                tc_fence_after();
                if (r == 0 && n < 8) V3_TR(k, (h == 0 ? 1 + n : 28));
                const uint32_t sb = tmem + lane_base + TM_SP0 + (uint32_t)b * 128 + (uint32_t)h * 64;
                uint32_t sr[64];
                float mx = -INFINITY;
#ifdef SLA2_ABL_NOSM
                if (false) {
#else
                if (has) {
#endif
#ifdef SLA2_ABL_NOSLD
#pragma unroll
                    for (int c = 0; c < 64; ++c) sr[c] = __float_as_uint(0.01f * (float)((c * 7 + r + n) & 31));
#else
                    tmem_ld32(sb, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                    tmem_ld32(sb + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                    tmem_ld_wait();
#endif
                    if (tail_kept && j == nb - 1) {  // ragged N: keys past N in the partial last block
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
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * p.scale_log2;
                }
                if (n == 0) {
                    sXch[h][r] = mx;
                    named_bar_sync(bar_x, 64);
                    m = fmaxf(mx, sXch[h ^ 1][r]);
                } else if (bar_red_or(bar_r, 64, mx > m + RESCALE_LOG2)) {
                    // either half of some row of this quarter grew past the lazy threshold: agree
                    // on the new maxima, then rescale this half's 64 O columns once PV(n-1) is in
                    sXch[h][r] = mx;
                    named_bar_sync(bar_x, 64);
                    const float mnew = fmaxf(m, fmaxf(mx, sXch[h ^ 1][r]));
                    const float corr = v3_exp2(m - mnew);
                    V3_WAIT(&bar_pv_done[(gg - 1) & 1], (uint32_t)(((gg - 1) >> 1) & 1));
                    __syncwarp();
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        uint32_t o[32];
                        const uint32_t oa = tmem + lane_base + TM_O + (uint32_t)h * 64 + c0;
                        tmem_ld32(oa, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * corr);
                        tmem_st32(oa, o);
                    }
                    l *= corr;
                    m = mnew;
                }
#ifdef SLA2_ABL_NOSM
                if (false) {
#else
                if (has) {
#endif
                    const float2 nm2 = make_float2(-m, -m);
                    float2 rs = make_float2(0.f, 0.f);
                    uint32_t w[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])),
                                                    sc2, nm2);
#ifdef SLA2_ABL_NOEXP
                        const float2 pe = __ffma2_rn(x, make_float2(0.001f, 0.001f), make_float2(0.5f, 0.5f));
#else
                        const float2 pe = make_float2(v3_exp2(x.x), v3_exp2(x.y));
#endif
                        rs = __fadd2_rn(rs, pe);
                        w[e] = pack_bf16(pe.x, pe.y);
                    }
                    tmem_st32(sb, w);  // P over this block's own S columns
                    l += rs.x + rs.y;
                    tmem_st_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_p_full[b]);
                if (r == 0 && h == 0 && n < 8) V3_TR(k, 9 + n);
            }
            // tile end: row sums to the epilogue; the barrier also retires this tile's exchanges
            named_bar_sync(bar_x, 64);
            if (r == 0 && h == 0) V3_TR(k, 31);
            if (k >= 1) V3_WAIT(&bar_l_free, (uint32_t)((k - 1) & 1));
            sLp[h][r] = l;
            mbar_arrive(&bar_sm_done);
            g += npair;
        }
    } else {
        v3_reg_alloc<176>();
        // ============ epilogue of tile k (thread = row r), concurrent with tile k+1 ============
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int gv = 0;
        int k = 0;
        for (int t = blockIdx.x; t < nt; t += G, ++k) {
            const V3Tile T = v3_tile(p, t);
            const int vhc = gv + T.nb;  // the tile's Hc slot
            const int hcs = vhc % NSV;
            gv = vhc + 1;
            const int64_t grow = T.bh * (int64_t)p.N + (int64_t)T.i * BQ + r;
            const bool row_live = T.i * BQ + r < p.N;  // ragged N: the last block's rows past N
            float alpha = 1.0f, bl = 0.0f;
            const uint4* ht = reinterpret_cast<const uint4*>(p.htot16 + (T.bh * D + r) * D);  // Htot row f = r
            if (T.linear) {
                // Htot row r into L1 now; it is read chunk by chunk while Hc is formed
                asm volatile("prefetch.global.L1 [%0];" ::"l"(ht));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(ht + 8));
                // den = phi(Q)_r . Zc (the bf16 phi(Q) the MMA uses)
                uint4 pq[16];
                const uint4* pqg = reinterpret_cast<const uint4*>(p.phiq + grow * D);
#pragma unroll
                for (int u = 0; u < 16; ++u) pq[u] = row_live ? pqg[u] : make_uint4(0u, 0u, 0u, 0u);
                // alpha = sigmoid(rho_i) with the reference's clamp (attention.hpp:17-22)
                const float x = p.rho[(int64_t)(T.bh % p.H) * p.tm + T.i];
                const float a = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x)));
                alpha = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
                V3_WAIT(&bar_zc_ready, (uint32_t)(k & 1));
                float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const uint32_t wv[4] = {pq[u].x, pq[u].y, pq[u].z, pq[u].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
                        d2 = __ffma2_rn(f2, *reinterpret_cast<const float2*>(&sZc[u * 8 + 2 * e]), d2);
                    }
                }
                const float den = d2.x + d2.y;
                bl = (row_live && den > 0.0f) ? (1.0f - alpha) / den : 0.0f;
            } else {
                V3_WAIT(&bar_zc_ready, (uint32_t)(k & 1));
            }
            mbar_arrive(&bar_zc_free);
            if (r == 0) V3_TR(k, 29);
            V3_WAIT(&bar_sm_done, (uint32_t)(k & 1));
            if (r == 0) V3_TR(k, 30);
            const float l = sLp[0][r] + sLp[1][r];
            mbar_arrive(&bar_l_free);
            const float al = alpha / l;
            // O -> registers as packed bf16 (alpha / l) O, then O's columns go to the next tile
            V3_WAIT(&bar_tile_done, (uint32_t)(k & 1));
            __syncwarp();
            tc_fence_after();
            if (r == 0) V3_TR(k, 17);
            uint32_t os[64];
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t o[32];
                tmem_ld32(tmem + lane_base + TM_O + c0, o);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    os[c0 / 2 + e] = pack_bf16(__uint_as_float(o[2 * e]) * al, __uint_as_float(o[2 * e + 1]) * al);
            }
            tc_fence_before();
            mbar_arrive(&bar_o_free);
            if (r == 0) V3_TR(k, 18);
            if (T.linear) {
                // Hc = Htot - Hsel, row f = r, as the MN-major B tile [c_atom 2][f 128][64 c] (bf16)
                V3_WAIT(&bar_v_full[hcs], (uint32_t)((vhc / NSV) & 1));  // the Hc slot is ours
                const uint32_t hb = smem_u32(sV(hcs));
#pragma unroll
                for (int c0 = 0; c0 < 128; c0 += 32) {
                    uint32_t hs[32];
                    uint4 hv4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) hv4[u] = ht[c0 / 8 + u];
                    tmem_ld32(tmem + lane_base + TM_H + c0, hs);
                    tmem_ld_wait();
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        const int c = c0 + ch * 8;
                        const uint32_t* t8 = reinterpret_cast<const uint32_t*>(&hv4[ch]);
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
                fence_proxy_async_smem();  // Hc is read by the async proxy
            }
            tc_fence_before();
            mbar_arrive(&bar_lin_ready);
            if (r == 0) V3_TR(k, 19);
            V3_WAIT(&bar_lin_done, (uint32_t)(k & 1));
            __syncwarp();
            tc_fence_after();
            if (r == 0) V3_TR(k, 20);
            // out = (alpha / l) O + ((1 - alpha) / den) phi(Q) Hc, row r (256 contiguous bytes)
            uint4* orow = reinterpret_cast<uint4*>(p.out + grow * D);
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t lv[32];
                if (T.linear) {
                    tmem_ld32(tmem + lane_base + TM_H + c0, lv);
                    tmem_ld_wait();
                }
                uint32_t w[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    float2 o2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&os[c0 / 2 + e]));
                    if (T.linear)
                        o2 = __ffma2_rn(make_float2(__uint_as_float(lv[2 * e]), __uint_as_float(lv[2 * e + 1])),
                                        make_float2(bl, bl), o2);
                    w[e] = pack_bf16(o2.x, o2.y);
                }
                if (row_live) {
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch)
                        orow[c0 / 8 + ch] = make_uint4(w[4 * ch], w[4 * ch + 1], w[4 * ch + 2], w[4 * ch + 3]);
                }
            }
            tc_fence_before();
            mbar_arrive(&bar_hl_free);  // the next tile's Hsel may overwrite the linear product
            if (r == 0) V3_TR(k, 21);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

bool sparse_v3_eligible(const SparseLaunch& a) {
    return !a.dense && a.bq == 128 && a.bk == 64 && a.d == 128 && a.o_s == nullptr && a.o_l == nullptr &&
           a.big_l == nullptr && a.h_blocks == nullptr && a.z_blocks == nullptr && a.phiq != nullptr &&
           a.tm_phiq != nullptr;
}

cudaError_t launch_sparse_v3(const SparseLaunch& a, cudaStream_t st, int* launches) {
    SparseV3Params p;
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
    p.last_valid = a.N - (a.tn - 1) * v3::BK;
    p.scale_log2 = a.inv_sqrt_d * 1.4426950408889634f;
#ifdef SLA2_TRACE
    extern unsigned long long* g_trace_buf;
    p.trace = g_trace_buf;
#endif
    cudaError_t e = ensure_smem_attr((const void*)sla2_sparse_v3_kernel, (int)v3::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = p.ntiles < sms ? p.ntiles : sms;
    sla2_sparse_v3_kernel<<<grid, v3::NTHREADS, v3::SMEM_BYTES, st>>>(*a.tm_q, *a.tm_k, *a.tm_v, *a.tm_phik,
                                                                      *a.tm_phiq, p);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
