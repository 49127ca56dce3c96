// sparse_v2.cu -- the persistent SLA2 sparse + linear + alpha-blend forward (sm_100a, bf16).
//
// Same algorithm as sparse_bf16.cu (the per-query-block loop of sla2_forward_blockwise,
// attention.hpp:484-558, with block_scores_qk / block_product_pv, 372-415), restructured so
// that one query block's epilogue and the next one's prologue run UNDER the neighbouring
// key-block loops instead of between them:
//
//  * persistent CTAs (one per SM) walk the (b, h, query block) tiles round robin;
//  * three warpgroups: WG0 = TMA producers (Q / K pairs / phi(Q); V / phi(K~) ring), the MMA
//    issuer and the Zc warp; WG1 = softmax (thread per query row) of tile k; WG2 = epilogue
//    (thread per row) of tile k-1, concurrently; setmaxnreg moves registers to WG1/WG2;
//  * one Q buffer: Q of tile k+1 loads as soon as tile k's last Q K^T has read it (it arrives
//    while tile k's last pairs and epilogue run); phi(Q) goes to TMEM, the output straight to
//    global, and the epilogue's Hc (Htot - Hsel, bf16) takes one V / phi(K~) ring slot per tile;
//  * the linear branch lands in the sparse accumulator: with c_r = (1 - a) l_r / (a den_r),
//        out = a / l (O + (c phi(Q)) (Htot - Hsel))
//    so the epilogue scales the phi(Q) rows by c, one MMA accumulates (c phi(Q)) Hc into O, and
//    O is read from TMEM once (attention.hpp:532-557: O_s = O / l, O_l = phi(Q) Hc / den,
//    out = a O_s + (1 - a) O_l);
//  * TMEM (512 columns): S 128 | P 2 x 64 | O 128 | Hsel 128. The epilogue of tile k reads
//    Hsel (then frees it for tile k+1's first phi(K~)^T V) and O (then frees it for tile k+1's
//    first PV); tile k+1's first Q K^T and softmax run meanwhile.
//
// Key blocks are processed in pairs (S = Q [K_2p; K_2p+1]^T, M128 N128 K128) exactly as in
// sparse_bf16.cu; see the comments there for the per-pair pipeline. The saved-state outputs
// (O_s, O_l, L, H_i, Z_i) and the dense mode stay on sparse_bf16.cu.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "expf_glibc.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace sla2dev {

namespace v2 {
constexpr int BQ = 128, BK = 64, D = 128;
// one Q buffer (the next tile's Q loads once this tile's last Q K^T is done), a ring of two K pairs
// and four V / phi(K~) slots (one per tile holds the epilogue's Hc). A second Q buffer instead of
// the 4th slot measured slower: the kernel waits on gather latency, so ring depth pays more
constexpr int NKP = 2, NSV = 4;
constexpr uint32_t Q_BYTES = BQ * D * 2;       // 32 KB
constexpr uint32_t TILE_BYTES = BK * D * 2;    // 16 KB
constexpr uint32_t TILE8_BYTES = BK * D;       // 8 KB: an E4M3 V / phi(K~) block (FP8 P/V mode)
constexpr uint32_t KP_BYTES = 2 * TILE_BYTES;  // a K pair
constexpr uint32_t VS_BYTES = 2 * TILE_BYTES;  // V + phi(K~), or Hc (bf16 128 x 128)
constexpr uint32_t OFF_Q = 0;                  // the Q buffer
constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
constexpr uint32_t OFF_V = OFF_K + NKP * KP_BYTES;
constexpr uint32_t SMEM_BYTES = OFF_V + NSV * VS_BYTES;  // 224 KB
constexpr uint32_t SMEM_ALLOC = SMEM_BYTES;  // + 3 KB static = the 227 KB limit: no alignment slack
constexpr uint32_t TM_S = 0, TM_P = 128, TM_O = 256, TM_H = 384;
constexpr float RESCALE_LOG2 = 8.0f;
constexpr int NTHREADS = 384;
}  // namespace v2

struct SparseV2Params {
    const int32_t* kv_idx;
    const int32_t* kv_cnt;
    int kstride, kappa;
    const float* rho;
    const float* ztot;
    const float* zblk;
    const __nv_bfloat16* htot16;  // [BH][D][D] bf16 (the epilogue forms Hc = Htot - Hsel from it)
    const __nv_bfloat16* phiq;    // [BH][N][D] bf16 phi(Q) rows (router front)
    __nv_bfloat16* out;           // [BH][N][D]
    const uint32_t* vamax;        // FP8 P/V mode: [BH] max |V| bits (V8 = e4m3(V * 448 / amax), phi8 = e4m3(448 phi))
    int N, H, tm, tn, ntiles;
    int last_valid;
    float scale_log2;
#ifdef SLA2_TRACE
    unsigned long long* trace;  // [grid][8 tiles][32 events] %globaltimer stamps (analysis build)
#endif
};

__device__ __forceinline__ float v2_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <uint32_t N>
__device__ __forceinline__ void reg_alloc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void reg_dealloc() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

// Bounded waits in analysis builds (-DSLA2_V2_WATCHDOG): a wait that spins ~seconds records
// (block, warp, site, parity) in g_v2_hang and traps instead of hanging the GPU.
#ifdef SLA2_V2_WATCHDOG
__device__ unsigned long long g_v2_hang[4];
__device__ __forceinline__ void v2_wait(uint64_t* bar, uint32_t parity, int site) {
    for (long long it = 0; !mbar_try_wait(bar, parity); ++it) {
        if (it == (1ll << 26)) {
            g_v2_hang[0] = blockIdx.x;
            g_v2_hang[1] = threadIdx.x >> 5;
            g_v2_hang[2] = (unsigned long long)site;
            g_v2_hang[3] = parity;
            __threadfence_system();
            printf("sla2_sparse_v2 HANG block %d warp %d lane %d line %d parity %u\n", blockIdx.x, threadIdx.x >> 5,
                   threadIdx.x & 31, site, parity);
            __trap();
        }
    }
}
#define V2_WAIT(bar, par) v2_wait(bar, par, __LINE__)
#else
#define V2_WAIT(bar, par) mbar_wait(bar, par)
#endif

#ifdef SLA2_TRACE
__device__ __forceinline__ unsigned long long v2_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// event e of this CTA's k-th tile (k < 8)
#define V2_TR(k, e) \
    if ((k) < 8) p.trace[((size_t)blockIdx.x * 8 + (k)) * 32 + (e)] = v2_gtimer()
#else
#define V2_TR(k, e)
#endif

// Everything about tile t every role needs (all roles walk the same tile sequence).
struct V2Tile {
    int64_t bh;
    int i, nb, npair;
    bool linear;
    const int32_t* idx;
};
__device__ __forceinline__ V2Tile v2_tile(const SparseV2Params& p, int t) {
    V2Tile r;
    r.bh = t / p.tm;
    r.i = t - (int)r.bh * p.tm;
    r.nb = p.kv_cnt ? p.kv_cnt[r.bh * p.tm + r.i] : p.kappa;
    r.npair = (r.nb + 1) >> 1;
    r.linear = r.nb != p.tn;
    r.idx = p.kv_idx + (r.bh * p.tm + r.i) * (int64_t)p.kstride;
    return r;
}

// MMA-issuer steps (whole warp; elect.sync inside each tcgen05 op). Plain functions with
// by-value state: the counters stay in registers (lambdas capturing them by reference put them
// on the stack).
__device__ __forceinline__ void v2_issue_qk(uint64_t* s_free, uint64_t* k_full, uint64_t* k_empty, uint64_t* s_full,
                                            int gg, uint32_t sbase, uint32_t tm, int nbu, int n) {
    using namespace v2;
    if (gg > 0) {
        V2_WAIT(s_free, (uint32_t)((gg - 1) & 1));  // S of pair gg-1 is in the softmax's registers
        tc_fence_after();
    }
    const int s = gg % NKP;
    V2_WAIT(&k_full[s], (uint32_t)((gg / NKP) & 1));
    tc_fence_after();
    const uint32_t idq = (2 * n + 1 < nbu) ? idesc_bf16(128, 128, false, false) : idesc_bf16(128, 64, false, false);
    const uint64_t dQ = sdesc_sw128(sbase + OFF_Q, 16, 1024);
    const uint64_t dK = sdesc_sw128(sbase + OFF_K + s * KP_BYTES, 16, 1024);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
        umma_bf16_ss_w(tm + TM_S, dQ + off, dK + off, idq, ks > 0);
    }
    umma_commit_w(s_full);
    umma_commit_w(&k_empty[s]);
}
// O += (c phi(Q)) Hc of tile kk once the epilogue has built both operands: A = c phi(Q) rows in
// the first 64 Hsel columns of TMEM (TS), B = Hc (MN-major) in the tile's Hc slot. The tile's
// Hsel was read before, and the next tile's phi(K~)^T V MMAs follow this one in the tensor pipe.
__device__ __forceinline__ void v2_lin_mma(uint64_t* lin_ready, uint64_t* lin_done, int kk, bool linear, int hc,
                                           uint32_t sbase, uint32_t tm) {
    using namespace v2;
    V2_WAIT(lin_ready, (uint32_t)(kk & 1));
    tc_fence_after();
    if (linear) {
        const uint64_t dB = sdesc_sw128(sbase + OFF_V + hc * VS_BYTES, 16384, 1024);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
            umma_bf16_ts_w(tm + TM_O, tm + TM_H + ks * 8, dB + ((ks * 2048) >> 4), idesc_bf16(128, 128, false, true), 1);
    }
    umma_commit_w(lin_done);
}

template <bool F8>
__global__ void __launch_bounds__(384, 1)
    sla2_sparse_v2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmPhi,
                          const SparseV2Params p) {
    using namespace v2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;  // 1024-aligned (static shared memory is a multiple of 1 KB; checked below)
    __shared__ uint64_t bar_q_full[2], bar_qk_done[2], bar_k_full[NKP],
        bar_k_empty[NKP], bar_v_full[NSV], bar_v_empty[NSV], bar_s_full, bar_s_free, bar_p_full[2], bar_pv_done[2],
        bar_tile_done, bar_sm_done[2], bar_lin_ready, bar_lin_done, bar_o_free, bar_zc_ready[2],
        bar_zc_free[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ float sZc[2][D];
    __shared__ float sL[2][BQ];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = p.ntiles, G = gridDim.x;
    auto sQ = [&](int) { return smem + OFF_Q; };
    auto sKp = [&](int s) { return smem + OFF_K + s * KP_BYTES; };
    auto sV = [&](int s) { return smem + OFF_V + s * VS_BYTES; };

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();  // SW128 tiles need 1 KB alignment
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_q_full[b], 1);
            mbar_init(&bar_qk_done[b], 1);
            mbar_init(&bar_p_full[b], 128);
            mbar_init(&bar_pv_done[b], 1);
            mbar_init(&bar_sm_done[b], 128);
            mbar_init(&bar_zc_ready[b], 1);
            mbar_init(&bar_zc_free[b], 128);
        }
        for (int s = 0; s < NKP; ++s) {
            mbar_init(&bar_k_full[s], 1);
            mbar_init(&bar_k_empty[s], 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(&bar_v_full[s], 1);
            mbar_init(&bar_v_empty[s], 1);
        }
        mbar_init(&bar_s_full, 1);
        mbar_init(&bar_s_free, 128);
        mbar_init(&bar_tile_done, 1);
        mbar_init(&bar_lin_ready, 128);
        mbar_init(&bar_lin_done, 1);
        mbar_init(&bar_o_free, 128);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(&tmem_base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    // register budget per thread: 72 (producers, MMA, Zc) + 224 (softmax) + 208 (epilogue) = 504 =
    // 3 x 168, the CTA's launch allocation (setmaxnreg.inc can only take what .dec released)
    if (warp < 4) {
        reg_dealloc<72>();
        if (warp == 0) {
            // ============ TMA producer: Q (two buffers), K pairs ============
            // one box per lane: bulk-tensor copies issued by one thread complete one after another
            if (lane == 0) {
                tma_prefetch_desc(&tmQ);
                tma_prefetch_desc(&tmK);
            }
            const uint64_t pol = policy_evict_last();
            auto load_q = [&](uint64_t* bar, uint8_t* dst, int qrow, int hz) {
                if (lane == 0) mbar_arrive_expect_tx(bar, Q_BYTES);
                __syncwarp();
                if (lane < 4) tma_load_3d(dst + lane * 8192, &tmQ, (lane >> 1) * 64, qrow + (lane & 1) * 64, hz, bar);
            };
            int64_t gk = 0;
            int t = blockIdx.x;
            if (t < nt) {
                const V2Tile T0 = v2_tile(p, t);
                load_q(&bar_q_full[0], sQ(0), T0.i * BQ, (int)T0.bh);
            }
            for (int k = 0; t < nt; ++k, t += G) {
                const V2Tile T = v2_tile(p, t);
                for (int n = 0; n < T.npair; ++n, ++gk) {
                    const int s = (int)(gk % NKP);
                    const int cnt = min(2, T.nb - 2 * n);
                    if (lane == 0) {
                        if (gk >= NKP) V2_WAIT(&bar_k_empty[s], (uint32_t)(((gk / NKP) - 1) & 1));
                        mbar_arrive_expect_tx(&bar_k_full[s], cnt * TILE_BYTES);
                    }
                    __syncwarp();
                    if (lane < 2 * cnt) {  // lane = (block b, 64-column half c)
                        const int b = lane >> 1, c = lane & 1;
                        const int krow = T.idx[2 * n + b] * BK;
                        tma_load_3d_hint(sKp(s) + c * 16384 + b * 8192, &tmK, c * 64, krow, (int)T.bh, &bar_k_full[s], pol);
                    }
                }
                // Q of the next tile, once tile k's last Q K^T has read the buffer
                if (t + G < nt) {
                    const V2Tile T1 = v2_tile(p, t + G);
                    const int k1 = k + 1;
                    if (lane == 0) V2_WAIT(&bar_qk_done[k & 1], (uint32_t)((k >> 1) & 1));  // tile k's last Q K^T
                    load_q(&bar_q_full[k1 & 1], sQ(k1 & 1), T1.i * BQ, (int)T1.bh);
                }
            }
        } else if (warp == 2) {
            // ============ TMA producer: V / phi(K~) ring; one slot per tile for the epilogue's Hc ============
            if (lane == 0) {
                tma_prefetch_desc(&tmV);
                tma_prefetch_desc(&tmPhi);
            }
            const uint64_t pol = policy_evict_last();
            int64_t gv = 0;
            for (int t = blockIdx.x; t < nt; t += G) {
                const V2Tile T = v2_tile(p, t);
                // FP8: one slot per key-block PAIR (V8 | phi8 of block 2n at 0 / 8 KB, of 2n+1 at
                // 16 / 24 KB), so the ring holds twice the blocks in flight; bf16: one per block
                const int nslot = F8 ? T.npair : T.nb;
                for (int j = 0; j <= nslot; ++j, ++gv) {
                    const int s = (int)(gv % NSV);
                    const int cnt = F8 ? min(2, T.nb - 2 * j) : 1;
                    if (lane == 0) {
                        if (gv >= NSV) V2_WAIT(&bar_v_empty[s], (uint32_t)(((gv / NSV) - 1) & 1));
                        if (j == nslot)  // the Hc slot: allocated, not loaded
                            mbar_arrive(&bar_v_full[s]);
                        else if (F8)
                            mbar_arrive_expect_tx(&bar_v_full[s], cnt * (T.linear ? 2 * TILE8_BYTES : TILE8_BYTES));
                        else
                            mbar_arrive_expect_tx(&bar_v_full[s], T.linear ? 2 * TILE_BYTES : TILE_BYTES);
                    }
                    __syncwarp();
                    if (F8) {  // one 128-byte-wide box per (block b, tensor t): lane = 2 b + t
                        const int b = lane >> 1, tt = lane & 1;
                        if (j < nslot && b < cnt && (tt == 0 || T.linear))
                            tma_load_3d_hint(sV(s) + b * TILE_BYTES + tt * TILE8_BYTES, tt == 0 ? &tmV : &tmPhi, 0,
                                             T.idx[2 * j + b] * BK, (int)T.bh, &bar_v_full[s], pol);
                    } else if (j < T.nb && lane < (T.linear ? 4 : 2)) {  // lane = (tensor V / phi, 64-column half)
                        const int krow = T.idx[j] * BK, hz = (int)T.bh, c = lane & 1;
                        tma_load_3d_hint(sV(s) + (lane >> 1) * TILE_BYTES + c * 8192, lane < 2 ? &tmV : &tmPhi, c * 64, krow,
                                         hz, &bar_v_full[s], pol);
                    }
                }
            }
        } else if (warp == 1) {
            // ============ MMA issuer (whole warp; elect.sync inside each tcgen05 op) ============
            constexpr uint32_t ID_QK2 = idesc_bf16(128, 128, false, false);
            constexpr uint32_t ID_QK1 = idesc_bf16(128, 64, false, false);
            constexpr uint32_t ID_PV = idesc_bf16(128, 128, false, true);
            constexpr uint32_t ID_HS = idesc_bf16(128, 128, true, true);
            constexpr uint32_t ID_LIN = idesc_bf16(128, 128, false, true);
            constexpr uint32_t ID_PV8 = idesc_e4m3(128, 128, false, true);
            constexpr uint32_t ID_HS8 = idesc_e4m3(128, 128, true, true);
            const uint32_t tm = warp_uniform(tmem);
            const uint32_t sbase = warp_uniform(smem_u32(smem));
            uint64_t* bar_s_free_p = &bar_s_free;
            const uint64_t dVm = sdesc_sw128(sbase + OFF_V, 8192, 1024);
            int g = 0, gv = 0;  // global pair / V-slot counters (< 2^31 per CTA)
            int k = 0;
            bool prev_linear = false;
            int prev_hc = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V2Tile T = v2_tile(p, t);
                const int nbu = (int)warp_uniform((uint32_t)T.nb);
                const int npu = (nbu + 1) >> 1;
                const bool lin = T.linear;
                const int pb = k & 1;
                V2_WAIT(&bar_q_full[pb], (uint32_t)((k >> 1) & 1));
                tc_fence_after();
                if (lane == 0) V2_TR(k, 0);
                v2_issue_qk(bar_s_free_p, bar_k_full, bar_k_empty, &bar_s_full, g, sbase, tm, nbu, 0);
                if (npu == 1) umma_commit_w(&bar_qk_done[pb]);
                for (int n = 0; n < npu; ++n) {
                    const int gg = g + n;
                    // tile k-1's linear term ahead of QK(1) in the tensor pipe: O (and the Hc slot) free
                    // sooner for PV(0); S(1) is not needed before P(0) anyway (measured 0.582 -> 0.566 ms)
                    if (n == 0 && k > 0)
                        v2_lin_mma(&bar_lin_ready, &bar_lin_done, k - 1, prev_linear, prev_hc, sbase, tm);
                    if (n + 1 < npu) {
                        v2_issue_qk(bar_s_free_p, bar_k_full, bar_k_empty, &bar_s_full, gg + 1, sbase, tm, nbu, n + 1);
                        if (n + 2 == npu) umma_commit_w(&bar_qk_done[pb]);  // the tile's last Q K^T
                    }
                    V2_WAIT(&bar_p_full[gg & 1], (uint32_t)((gg >> 1) & 1));
                    tc_fence_after();
                    if (n == 0 && k > 0) {
                        V2_WAIT(&bar_o_free, (uint32_t)((k - 1) & 1));  // tile k-1's O left TMEM
                        tc_fence_after();
                    }
                    if (lane == 0 && n < 8) V2_TR(k, 25 + (n < 2 ? n : 2));
                    const int j0 = 2 * n, j1 = min(nbu, j0 + 2);
                    if (F8) {  // the pair's slot
                        const int v = gv + n;
                        V2_WAIT(&bar_v_full[v % NSV], (uint32_t)((v / NSV) & 1));
                        tc_fence_after();
                    }
                    for (int j = j0; j < j1; ++j) {
                        const int v = F8 ? gv + n : gv + j;
                        const int sv = v % NSV;
                        if (!F8) {
                            V2_WAIT(&bar_v_full[sv], (uint32_t)((v / NSV) & 1));
                            tc_fence_after();
                        }
                        const uint64_t dV = dVm + ((sv * VS_BYTES + (F8 ? (j & 1) * TILE_BYTES : 0)) >> 4);
                        if (F8) {  // P: 4 e4m3 per TMEM column (16 per key block); V8 MN-major, 32 keys per MMA
                            const uint32_t aP = tm + TM_P + (uint32_t)((gg & 1) * 64 + (j & 1) * 16);
#pragma unroll
                            for (int ks = 0; ks < 2; ++ks)
                                umma_f8_ts_w(tm + TM_O, aP + ks * 8, dV + ((ks * 4096) >> 4), ID_PV8, (j > 0 || ks > 0));
                        } else {
                            const uint32_t aP = tm + TM_P + (uint32_t)((gg & 1) * 64 + (j & 1) * 32);
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                umma_bf16_ts_w(tm + TM_O, aP + ks * 8, dV + ((ks * 2048) >> 4), ID_PV, (j > 0 || ks > 0));
                        }
                    }
                    umma_commit_w(&bar_pv_done[gg & 1]);
                    for (int j = j0; j < j1; ++j) {
                        const int sv = (int)((F8 ? gv + n : gv + j) % NSV);
                        if (lin) {
                            const uint64_t dV = dVm + ((sv * VS_BYTES + (F8 ? (j & 1) * TILE_BYTES : 0)) >> 4);
                            const uint64_t dP = dV + ((F8 ? TILE8_BYTES : TILE_BYTES) >> 4);
                            if (F8) {
#pragma unroll
                                for (int ks = 0; ks < 2; ++ks)
                                    umma_f8_ss_w(tm + TM_H, dP + ((ks * 4096) >> 4), dV + ((ks * 4096) >> 4), ID_HS8,
                                                 (j > 0 || ks > 0));
                            } else {
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks)
                                    umma_bf16_ss_w(tm + TM_H, dP + ((ks * 2048) >> 4), dV + ((ks * 2048) >> 4), ID_HS,
                                                   (j > 0 || ks > 0));
                            }
                        }
                        if (!F8 || j == j1 - 1) umma_commit_w(&bar_v_empty[sv]);  // FP8: once per pair slot
                    }
                }
                umma_commit_w(&bar_tile_done);
                if (lane == 0) V2_TR(k, 28);
                g += npu;
                gv += F8 ? npu : nbu;
                prev_hc = gv % NSV;  // the tile's Hc slot
                gv += 1;
                prev_linear = lin;
            }
            if (k > 0) v2_lin_mma(&bar_lin_ready, &bar_lin_done, k - 1, prev_linear, prev_hc, sbase, tm);
        } else if (warp == 3) {
            // ============ Zc = Ztot - sum_sel z_j per tile (the linear denominators) ============
            int k = 0;
            for (int t = blockIdx.x; t < nt; t += G, ++k) {
                const V2Tile T = v2_tile(p, t);
                const int pb = k & 1;
                if (k >= 2) V2_WAIT(&bar_zc_free[pb], (uint32_t)(((k >> 1) - 1) & 1));
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
                    sZc[pb][lane * 4 + 0] = zt.x - acc.x;
                    sZc[pb][lane * 4 + 1] = zt.y - acc.y;
                    sZc[pb][lane * 4 + 2] = zt.z - acc.z;
                    sZc[pb][lane * 4 + 3] = zt.w - acc.w;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_zc_ready[pb]);
            }
        }
    } else if (warp < 8) {
        reg_alloc<224>();
        // ============ softmax: thread = query row r of tile k ============
        const int r = threadIdx.x - 128;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int64_t g = 0;
        int k = 0;
        for (int t = blockIdx.x; t < nt; t += G, ++k) {
            const V2Tile T = v2_tile(p, t);
            const int nb = T.nb, npair = T.npair;
            const bool tail_kept = p.last_valid < BK && T.idx[nb - 1] == p.tn - 1;
            float m2 = -INFINITY, l = 0.0f;
            for (int n = 0; n < npair; ++n) {
                const int64_t gg = g + n;
                const int b = (int)(gg & 1);
                const bool two = 2 * n + 1 < nb;
                V2_WAIT(&bar_s_full, (uint32_t)(gg & 1));
                __syncwarp();
                tc_fence_after();
                if (r == 0 && n < 8) V2_TR(k, 1 + n);
                const uint32_t sbase = tmem + lane_base + TM_S;
                if (tail_kept && n == npair - 1) {
                    // ragged N: keys past N in the partial last key block get -inf (see sparse_bf16.cu)
                    const uint32_t col0 = (uint32_t)(((nb - 1) - 2 * n) * 64);
                    for (int tt = p.last_valid; tt < BK; ++tt) tmem_st1(sbase + col0 + tt, __float_as_uint(-INFINITY));
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
                mbar_arrive(&bar_s_free);
                float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int tt = 0; tt < 64; tt += 8) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        m4[u] = fmaxf(m4[u], fmaxf(__uint_as_float(sr[tt + 2 * u]), __uint_as_float(sr[tt + 2 * u + 1])));
                }
                if (two) {
#pragma unroll
                    for (int tt = 64; tt < 128; tt += 8) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            m4[u] = fmaxf(m4[u],
                                          fmaxf(__uint_as_float(sr[tt + 2 * u]), __uint_as_float(sr[tt + 2 * u + 1])));
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
                        const float corr = v2_exp2(m2 - mnew);
                        V2_WAIT(&bar_pv_done[(gg - 1) & 1], (uint32_t)(((gg - 1) >> 1) & 1));  // PVs so far
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
                if (gg >= 2) {  // P buffer b was last read by PV(gg - 2)
                    V2_WAIT(&bar_pv_done[b], (uint32_t)(((gg - 2) >> 1) & 1));
                    __syncwarp();
                    tc_fence_after();
                }
                const uint32_t pbase = tmem + lane_base + TM_P + b * 64;
                const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m2, -m2);
                float2 rs = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int blk = 0; blk < 2; ++blk) {
                    if (blk == 1 && !two) break;
                    if (F8) {  // P <= 2^RESCALE_LOG2 = 256 < 448: e4m3 without a scale, 4 keys per column
                        uint32_t w[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const float2 xa = __ffma2_rn(make_float2(__uint_as_float(sr[blk * 64 + 4 * e]),
                                                                     __uint_as_float(sr[blk * 64 + 4 * e + 1])),
                                                         sc2, nm2);
                            const float2 xb = __ffma2_rn(make_float2(__uint_as_float(sr[blk * 64 + 4 * e + 2]),
                                                                     __uint_as_float(sr[blk * 64 + 4 * e + 3])),
                                                         sc2, nm2);
                            const float2 pa = make_float2(v2_exp2(xa.x), v2_exp2(xa.y));
                            const float2 pb2 = make_float2(v2_exp2(xb.x), v2_exp2(xb.y));
                            rs = __fadd2_rn(rs, __fadd2_rn(pa, pb2));
                            w[e] = pack_e4m3x2(pa.x, pa.y) | (pack_e4m3x2(pb2.x, pb2.y) << 16);
                        }
                        tmem_st16(pbase + blk * 16, w);
                    } else {
                        uint32_t w[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) {  // packed FFMA2 / FADD2 (half the issue of scalar)
                            const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[blk * 64 + 2 * e]),
                                                                     __uint_as_float(sr[blk * 64 + 2 * e + 1])),
                                                         sc2, nm2);
                            const float2 pe = make_float2(v2_exp2(x2.x), v2_exp2(x2.y));
                            rs = __fadd2_rn(rs, pe);
                            w[e] = pack_bf16(pe.x, pe.y);
                        }
                        tmem_st32(pbase + blk * 32, w);
                    }
                }
                l += rs.x + rs.y;
                if (n == npair - 1) sL[k & 1][r] = l;  // before the last P: the epilogue's 1 / l
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&bar_p_full[b]);
                if (r == 0 && n < 8) V2_TR(k, 9 + n);
            }
            mbar_arrive(&bar_sm_done[k & 1]);
            g += npair;
        }
    } else {
        reg_alloc<208>();
        // ============ epilogue of tile k (thread = row r), one tile behind the softmax ============
        const int r = threadIdx.x - 256;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int gv = 0;
        int k = 0;
        for (int t = blockIdx.x; t < nt; t += G, ++k) {
            const V2Tile T = v2_tile(p, t);
            const int pb = k & 1;
            const int vhc = gv + (F8 ? T.npair : T.nb);  // the tile's Hc slot
            const int hcs = vhc % NSV;
            gv = vhc + 1;
            const int64_t grow = T.bh * (int64_t)p.N + (int64_t)T.i * BQ + r;
            const bool row_live = T.i * BQ + r < p.N;  // ragged N: the last block's rows past N
            float alpha = 1.0f, l = 1.0f;
            // FP8 P/V: O and Hsel accumulate in V8 units (V = vs V8, phi = phi8 / 448):
            // out = alpha / l * vs * (O8 + (c phi(Q)) Hc8), Hc8 = Htot / vs - Hsel8 / 448
            float vs = 1.0f, ivs = 1.0f;
            if (F8) {
                const float am = __uint_as_float(p.vamax[T.bh]);
                vs = am > 0.0f ? am * (1.0f / 448.0f) : 1.0f;
                ivs = 1.0f / vs;
            }
            const float hs_scale = F8 ? 1.0f / 448.0f : 1.0f;
            uint32_t cq[64];  // c phi(Q)_r as packed bf16 pairs (the lin MMA's A row)
            uint4 htr[16];    // Htot row f = r (bf16)
            if (T.linear) {
                // loads in flight first: Htot row r and phi(Q) row r (global / L2)
                const uint4* ht = reinterpret_cast<const uint4*>(p.htot16 + (T.bh * D + r) * D);
#pragma unroll
                for (int u = 0; u < 16; ++u) htr[u] = ht[u];
                const uint4* pq = reinterpret_cast<const uint4*>(p.phiq + grow * D);
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const uint4 w = row_live ? pq[u] : make_uint4(0u, 0u, 0u, 0u);
                    cq[4 * u] = w.x;
                    cq[4 * u + 1] = w.y;
                    cq[4 * u + 2] = w.z;
                    cq[4 * u + 3] = w.w;
                }
                // alpha = sigmoid(rho_i) with the reference's clamp (attention.hpp:17-22)
                const float x = p.rho[(int64_t)(T.bh % p.H) * p.tm + T.i];
                float a = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x)));
                alpha = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
                V2_WAIT(&bar_zc_ready[pb], (uint32_t)((k >> 1) & 1));
                if (r == 0) V2_TR(k, 29);
                float d4[4] = {0.f, 0.f, 0.f, 0.f};  // den = phi(Q)_r . Zc (the bf16 phi(Q) the MMA uses)
#pragma unroll
                for (int e = 0; e < 64; ++e) {
                    const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cq[e]));
                    d4[e & 3] = fmaf(f2.y, sZc[pb][2 * e + 1], fmaf(f2.x, sZc[pb][2 * e], d4[e & 3]));
                }
                const float den = (d4[0] + d4[1]) + (d4[2] + d4[3]);
                V2_WAIT(&bar_sm_done[pb], (uint32_t)((k >> 1) & 1));
                if (r == 0) V2_TR(k, 31);
                l = sL[pb][r];
                const float c = (row_live && den > 0.0f) ? (1.0f - alpha) * l / (alpha * den) : 0.0f;
#pragma unroll
                for (int e = 0; e < 64; ++e) {
                    const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cq[e]));
                    cq[e] = pack_bf16(f2.x * c, f2.y * c);
                }
            } else {
                V2_WAIT(&bar_sm_done[pb], (uint32_t)((k >> 1) & 1));
                l = sL[pb][r];
            }
            mbar_arrive(&bar_zc_free[pb]);
            V2_WAIT(&bar_tile_done, (uint32_t)(k & 1));  // every PV / phi(K~)^T V of the tile
            __syncwarp();
            tc_fence_after();
            if (r == 0) V2_TR(k, 17);
            if (T.linear) {
                // Hc = Htot - Hsel, row f = r, as the MN-major B tile [c_atom 2][f 128][64 c] (bf16)
                V2_WAIT(&bar_v_full[hcs], (uint32_t)((vhc / NSV) & 1));  // the Hc slot is ours
                const uint32_t hb = smem_u32(sV(hcs));
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
                            if (F8)
                                o4[e] = pack_bf16(tf.x * ivs - __uint_as_float(hs[ch * 8 + 2 * e]) * hs_scale,
                                                  tf.y * ivs - __uint_as_float(hs[ch * 8 + 2 * e + 1]) * hs_scale);
                            else
                                o4[e] = pack_bf16(tf.x - __uint_as_float(hs[ch * 8 + 2 * e]),
                                                  tf.y - __uint_as_float(hs[ch * 8 + 2 * e + 1]));
                        }
                        st_shared_v4(hb + (c >> 6) * 16384 + sw128_off(r, c & 63), o4[0], o4[1], o4[2], o4[3]);
                    }
                }
                // c phi(Q)_r into this lane's first 64 Hsel columns: the lin MMA's TMEM A operand
                tmem_st32(tmem + lane_base + TM_H, *reinterpret_cast<uint32_t(*)[32]>(&cq[0]));
                tmem_st32(tmem + lane_base + TM_H + 32, *reinterpret_cast<uint32_t(*)[32]>(&cq[32]));
                tmem_st_wait();
                fence_proxy_async_smem();  // Hc is read by the async proxy
            }
            tc_fence_before();
            mbar_arrive(&bar_lin_ready);
            if (r == 0) V2_TR(k, 19);
            V2_WAIT(&bar_lin_done, (uint32_t)(k & 1));
            __syncwarp();
            tc_fence_after();
            if (r == 0) {
                V2_TR(k, 20);
                mbar_arrive(&bar_v_empty[hcs]);  // the lin MMA has read Hc: the slot returns to the V ring
            }
            // out = alpha / l * O straight to global (row r: 256 contiguous bytes)
            const float sc = F8 ? alpha / l * vs : alpha / l;
            uint4* orow = reinterpret_cast<uint4*>(p.out + grow * D);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t o[64];
                tmem_ld32(tmem + lane_base + TM_O + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                tmem_ld32(tmem + lane_base + TM_O + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
                tmem_ld_wait();
                if (half == 1) {
                    tc_fence_before();
                    mbar_arrive(&bar_o_free);  // the next tile's first PV may overwrite O
                    if (r == 0) V2_TR(k, 21);
                }
                if (row_live) {
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch)
                        orow[half * 8 + ch] =
                            make_uint4(pack_bf16(__uint_as_float(o[ch * 8 + 0]) * sc, __uint_as_float(o[ch * 8 + 1]) * sc),
                                       pack_bf16(__uint_as_float(o[ch * 8 + 2]) * sc, __uint_as_float(o[ch * 8 + 3]) * sc),
                                       pack_bf16(__uint_as_float(o[ch * 8 + 4]) * sc, __uint_as_float(o[ch * 8 + 5]) * sc),
                                       pack_bf16(__uint_as_float(o[ch * 8 + 6]) * sc, __uint_as_float(o[ch * 8 + 7]) * sc));
                }
            }
            if (r == 0) V2_TR(k, 22);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

bool sparse_v2_eligible(const SparseLaunch& a) {
    return !a.dense && a.bq == 128 && a.bk == 64 && a.d == 128 && a.o_s == nullptr && a.o_l == nullptr &&
           a.big_l == nullptr && a.h_blocks == nullptr && a.z_blocks == nullptr && a.phiq != nullptr;
}

cudaError_t launch_sparse_v2(const SparseLaunch& a, cudaStream_t st, int* launches) {
    SparseV2Params p;
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
    p.vamax = a.vamax;
    p.N = a.N;
    p.H = (int)a.H;
    p.tm = a.tm;
    p.tn = a.tn;
    p.ntiles = (int)(a.B * a.H) * a.tm;
    p.last_valid = a.N - (a.tn - 1) * v2::BK;
    p.scale_log2 = a.inv_sqrt_d * 1.4426950408889634f;
#ifdef SLA2_TRACE
    extern unsigned long long* g_trace_buf;
    p.trace = g_trace_buf;
#endif
    const bool f8 = a.vamax != nullptr;
    const void* fn = f8 ? (const void*)sla2_sparse_v2_kernel<true> : (const void*)sla2_sparse_v2_kernel<false>;
    cudaError_t e = ensure_smem_attr(fn, (int)v2::SMEM_ALLOC);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = p.ntiles < sms ? p.ntiles : sms;
    if (f8)
        sla2_sparse_v2_kernel<true><<<grid, v2::NTHREADS, v2::SMEM_ALLOC, st>>>(*a.tm_q, *a.tm_k, *a.tm_v8, *a.tm_phi8, p);
    else
        sla2_sparse_v2_kernel<false><<<grid, v2::NTHREADS, v2::SMEM_ALLOC, st>>>(*a.tm_q, *a.tm_k, *a.tm_v, *a.tm_phik, p);
    ++*launches;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ FP8 P/V operand preparation
// (tolerance mode, not in the reference, which is INT8-only: quant.hpp:15-19). Per head one
// scale for V: amax = max |V| over the head's N x d entries (fp32 bits, atomicMax on the
// non-negative bit patterns), V8 = e4m3(V * 448 / amax); phi(K~) is a row softmax in (0, 1], so
// phi8 = e4m3(448 phi) needs no scale. Both are [BH][N][128] E4M3, the sparse kernel's
// 128-byte-wide TMA boxes.
__device__ __forceinline__ float absmax8_bf16(uint4 w) {
    float r = 0.0f;
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        r = fmaxf(r, fabsf(__uint_as_float(u[e] << 16)));
        r = fmaxf(r, fabsf(__uint_as_float(u[e] & 0xFFFF0000u)));
    }
    return r;
}
__global__ void __launch_bounds__(256) v_absmax_kernel(const uint4* __restrict__ v, uint32_t* __restrict__ amax,
                                                       int64_t per_head) {  // per_head: uint4 per head
    const int64_t bh = blockIdx.y;
    const uint4* src = v + bh * per_head;
    float m = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < per_head; i += (int64_t)gridDim.x * 256)
        m = fmaxf(m, absmax8_bf16(src[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = fmaxf(m, wm[w]);
        atomicMax(amax + bh, __float_as_uint(m));
    }
}
__device__ __forceinline__ uint2 e4m3x8(uint4 w, float s) {
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
    uint32_t r[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t a = u[2 * h], b = u[2 * h + 1];
        r[h] = pack_e4m3x2(__uint_as_float(a << 16) * s, __uint_as_float(a & 0xFFFF0000u) * s) |
               (pack_e4m3x2(__uint_as_float(b << 16) * s, __uint_as_float(b & 0xFFFF0000u) * s) << 16);
    }
    return make_uint2(r[0], r[1]);
}
// dst = e4m3(src * scale), scale = 448 / amax[head] (amax non-null) or `cscale`
__global__ void __launch_bounds__(256) e4m3_convert_kernel(const uint4* __restrict__ src, const uint32_t* __restrict__ amax,
                                                           float cscale, uint2* __restrict__ dst, int64_t per_head,
                                                           int64_t total) {
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
        float s = cscale;
        if (amax) {
            const float am = __uint_as_float(__ldg(amax + i / per_head));
            s = am > 0.0f ? 448.0f / am : 1.0f;
        }
        dst[i] = e4m3x8(src[i], s);
    }
}

// v non-null: amax = max |V| per head, then V8; phik non-null: phi8 = e4m3(448 phi(K~)).
cudaError_t launch_fp8pv_prep(const void* v, const void* phik, uint8_t* v8, uint8_t* phi8, uint32_t* amax, int64_t BH,
                              int64_t N, cudaStream_t st, int* launches) {
    const int64_t per_head = N * 128 / 8;  // uint4 (8 bf16) per head
    const int64_t total = BH * per_head;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    if (v) {
        cudaError_t e = cudaMemsetAsync(amax, 0, BH * sizeof(uint32_t), st);
        if (e != cudaSuccess) return e;
        const int gx = (int)std::min<int64_t>((per_head + 2047) / 2048, std::max<int64_t>(1, (int64_t)sms * 8 / BH + 1));
        v_absmax_kernel<<<dim3(gx, (unsigned)BH), 256, 0, st>>>((const uint4*)v, amax, per_head);
        ++*launches;
        e4m3_convert_kernel<<<grid, 256, 0, st>>>((const uint4*)v, amax, 1.0f, (uint2*)v8, per_head, total);
        ++*launches;
    }
    if (phik) {
        e4m3_convert_kernel<<<grid, 256, 0, st>>>((const uint4*)phik, nullptr, 448.0f, (uint2*)phi8, per_head, total);
        ++*launches;
    }
    return cudaGetLastError();
}

}  // namespace sla2dev
