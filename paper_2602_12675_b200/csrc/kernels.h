// kernels.h -- internal launch interface between the C ABI (capi.cu) and the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sla2dev {

// ---- per-device host state (capi.cu)
// Helper streams / events are cached per (thread, current device) and the >48 KB shared-memory
// attribute is set once per (device, kernel): a process that drives two GPUs never queues
// device-1 work on a device-0 stream nor launches on a device whose attribute was not set.
// `slot` names the call site; prio: +1 highest stream priority, -1 lowest, 0 default.
cudaStream_t aux_stream(int slot, int prio);
cudaEvent_t aux_event(int slot);
cudaError_t ensure_smem_attr(const void* func, int bytes);

// ---- router (router.cu)
struct RouterLaunch {
    const void* q;
    const void* k;
    bool bf16;
    int64_t B, H;
    int N, d, bq, bk, kappa;
    int smooth, exact_mu;
    float inv_sqrt_d;
    const float* proj_q;
    const float* proj_k;
    const CUtensorMap* tm_kcol;  // K as [B*H*N][d], box 32 cols x 256 rows, no swizzle (or null)
    float* mu_out;    // [BH][d] (written unless null)
    double* mu_part;  // fast colmean scratch
    float* qp;        // [BH][tm][d]
    float* kp;        // [BH][tn][d]
    float* qbar;      // [BH][tm][d] pooled scratch
    float* kbar;      // [BH][tn][d] pooled scratch
    float* pc_out;    // optional [BH][tm][tn]
    uint8_t* mask_out;
    int32_t* idx_out;  // [BH][tm][kappa]
    cudaEvent_t mu_ready;  // optional: recorded once mu_out is complete (lets the caller fork
                           // the linear-branch precompute off it)
    bool kbar_ready;       // kbar already holds the pooled keys (launch_kprep): back half only projects
    void* phiq_out;        // optional: the front half also writes phi(Q) here (launch_phiq, bf16 d = 128)
    cudaEvent_t query_done;  // optional: recorded once the query side is done (before the mu join)
};
// stage-timing hook (capi.cu): records timeline event `slot` on st when timing is enabled
void timeline_mark(int slot, cudaStream_t st);
cudaError_t launch_router(const RouterLaunch& a, cudaStream_t st, int* launches);
// The two halves of launch_router: front = mu (side stream, joined into st) + query-side
// pooling/projection; back = key-side pooling (unless kbar_ready)/projection + scores/top-k.
cudaError_t launch_router_front(const RouterLaunch& a, cudaStream_t st, int* launches);
cudaError_t launch_router_back(const RouterLaunch& a, cudaStream_t st, int* launches);
// parallel fp64 column mean (not the reference's serial order): the linear branch's mu
cudaError_t launch_colmean(const void* k, const CUtensorMap* tmk, bool bf16, float* mu, int BH, int N, int d,
                           cudaStream_t st, int* launches);
cudaError_t launch_topk_only(const float* pc, int BH, int tm, int tn, int kappa, uint8_t* mask, int32_t* idx,
                             cudaStream_t st, int* launches);
cudaError_t launch_mask_to_idx(const uint8_t* mask, int rows, int tn, int32_t* idx, int32_t* cnt, int* empty_flag,
                               cudaStream_t st, int* launches);

// ---- linear-branch precompute (linear.cu)
struct LinearLaunch {
    const void* k;
    const void* v;
    bool bf16;
    int64_t BH;
    int N, d, bk;
    const float* mu;  // null when smooth == 0
    void* phik;       // bf16 [BH][N][d] (bf16 path) or fp32 (f32 path)
    float* zblk;      // [BH][tn][d] colsum of (rounded) phi(K~) per key block
    float* ztot;      // [BH][d]
    float* hpart;     // [BH][nchunk][d][d] partial phi(K~)^T V
    float* htot;      // [BH][d][d]
    void* htot16;     // [BH][d][d] bf16 copy (bf16 path; the sparse kernel's TMA source)
    int nchunk;       // key-block chunks per head for the H partials
    const CUtensorMap* tm_phik;  // bf16 path: TMA maps (box 64x64, SW128) over [BH*N][d]
    const CUtensorMap* tm_v;
    const CUtensorMap* tm_k;  // bf16 path: K map (box 64x64, SW128); with mu set, phi(K~) is fused
                              // into the Htot partial kernel (kphi_htot_kernel)
    bool phik_ready;  // phi(K~) and z_j already written by launch_kprep
    uint8_t* phi8 = nullptr;  // FP8 P/V mode: the fused kernel writes E4M3 448 phi(K~) here instead of phik
};
cudaError_t launch_linear_prep(const LinearLaunch& a, cudaStream_t st, int* launches);
// Fused key-side prep (d = 128): phi(K~) + z_j (as phik_kernel) and the router's pooled keys
// kbar [BH][tn][d] (as pool_project_kernel's pooling), reading K once.
cudaError_t launch_kprep(const LinearLaunch& a, float* kbar, cudaStream_t st, int* launches);
// the two halves of launch_kprep: pooled keys only (router critical path) / phi(K~) and z_j only
cudaError_t launch_kpool(const LinearLaunch& a, float* kbar, cudaStream_t st, int* launches);
cudaError_t launch_kphi(const LinearLaunch& a, cudaStream_t st, int* launches);
// phi(Q) rows (bf16, d = 128) for the sparse kernel's linear-branch MMA: [rows][128] -> [rows][128]
cudaError_t launch_phiq(const void* q, void* phiq, int64_t rows, cudaStream_t st, int* launches);
// exact fp32 row softmax over d (SLA2ForwardSaved q_phi / k_phi; mu non-null: of K - mu)
cudaError_t launch_phi_exact(const void* x, bool bf16, const float* mu, float* out, int64_t rows, int N, int d,
                             cudaStream_t st, int* launches);

// ---- sparse / dense attention (sparse_bf16.cu, sparse_f32.cu)
struct SparseLaunch {
    int64_t B, H;
    int N, d, bq, bk, tm, tn;
    const int32_t* kv_idx;  // [BH][tm][kstride]
    const int32_t* kv_cnt;  // [BH][tm] or null (every row keeps `kappa`)
    int kstride, kappa;
    const float* rho;   // [H][tm]
    const float* htot;  // [BH][d][d]
    const void* htot16;  // [BH][d][d] bf16 copy (bf16 path)
    const float* ztot;  // [BH][d]
    const float* zblk;  // [BH][tn][d]
    const float* mu;    // [BH][d] (for L correction / f32 K~), may be null when smooth == 0
    int smooth;
    int dense;          // visit every key block, no linear branch (full_attention)
    float inv_sqrt_d;
    void* out;
    float* o_s;
    float* o_l;
    float* big_l;
    float* h_blocks;  // [BH][tm][d][d] complement H_i = sum of unselected h_j (saved path), or null
    float* z_blocks;  // [BH][tm][d] complement Z_i, or null
    float* s_first;   // QAT only: [BH][tm][bq][bk] S of each query block's first kept key block, or null
    // bf16 path
    const CUtensorMap* tm_q;
    const CUtensorMap* tm_k;
    const CUtensorMap* tm_v;
    const CUtensorMap* tm_phik;
    const CUtensorMap* tm_ht;  // Htot bf16 as [BH*d][d], box 64 x 128, SW128
    const CUtensorMap* tm_phiq;  // phi(Q) bf16 as [BH*N][d] (launch_phiq), box 64 x 64, SW128
    const void* phiq;            // the same phi(Q) rows (bf16 [BH][N][d])
    const CUtensorMap* tm_out;   // out bf16 as [BH*N][d], box 64 x 64, SW128 (TMA-stored blocks)
    void* ol;                    // bf16 [BH][N][d] scratch: the linear branch's O_l (sparse_fa.cu)
    // FP8 P/V mode (sparse_v2.cu, non-null vamax): E4M3 V8 / phi8 [BH][N][128] maps (box 128 x 64 B)
    const uint32_t* vamax;       // [BH] max |V| bits
    const CUtensorMap* tm_v8;
    const CUtensorMap* tm_phi8;
    // f32 path
    const float* q;
    const float* k;
    const float* v;
    const float* phik;
};
cudaError_t launch_sparse_bf16(const SparseLaunch& a, cudaStream_t st, int* launches);
// persistent variant (sparse_v2.cu): the non-saved, non-dense bf16 path
bool sparse_v2_eligible(const SparseLaunch& a);
cudaError_t launch_sparse_v2(const SparseLaunch& a, cudaStream_t st, int* launches);
// FP8 P/V operands: amax[bh] = max |V|, v8 = e4m3(V * 448 / amax), phi8 = e4m3(448 phi(K~)) (bf16 in)
cudaError_t launch_fp8pv_prep(const void* v, const void* phik, uint8_t* v8, uint8_t* phi8, uint32_t* amax, int64_t BH,
                              int64_t N, cudaStream_t st, int* launches);
// split forward (sparse_fa.cu): linear-branch kernel (O_l) + two-query-block attention kernel;
// also the dense mode (full_attention)
bool sparse_fa_eligible(const SparseLaunch& a);
cudaError_t launch_sparse_fa(const SparseLaunch& a, cudaStream_t st, int* launches);
// the linear branch alone: O_l = phi(Q) Hc / (phi(Q) . Zc) per query block into a.ol (bf16)
cudaError_t launch_linsel(const SparseLaunch& a, cudaStream_t st, int* launches);
cudaError_t launch_sparse_f32(const SparseLaunch& a, cudaStream_t st, int* launches);
size_t sparse_f32_smem_bytes(int d, int bq, int bk);

// ---- INT8 QAT path (quant.cu)
struct QuantLaunch {
    int64_t B, H;
    int N, d, bq, bk, tm, tn;
    const void* q;  // bf16
    const void* k;
    const void* v;
    const float* mu;
    int smooth;
    int8_t* qc;     // [BH][N][d] Q codes per query block
    float* qs;      // [BH][tm]
    int8_t* kc;     // [BH][N][d] K~ codes per key block
    float* ks;      // [BH][tn]
    int8_t* vct;    // [BH][N][d] V codes per key block (row-major, the PV MMA's MN-major B tile)
    float* vs;      // [BH][tn]
    int which = 7;  // tensors to quantize: 1 = Q, 2 = K~, 4 = V
};
cudaError_t launch_quant_prep(const QuantLaunch& a, cudaStream_t st, int* launches);
struct SparseI8Launch {
    SparseLaunch s;
    const int8_t* qc;
    const float* qs;
    const int8_t* kc;
    const float* ks;
    const int8_t* vct;
    const float* vs;
    const CUtensorMap* tm_qc;   // [BH*N][d] int8, box 128x128
    const CUtensorMap* tm_kc;   // [BH*N][d] int8, box 128(x) x 64(y)
    const CUtensorMap* tm_vct;  // [BH*N][d] int8, box 128 x 64
};
cudaError_t launch_sparse_i8(const SparseI8Launch& a, cudaStream_t st, int* launches);
// two-query-block INT8 attention (attn_i8.cu) after the bf16 linear-branch kernel; tm_phik3 /
// tm_v3 are the 3-D [BH][N][d] maps the linear-branch kernel reads
bool attn_i8_eligible(const SparseI8Launch& a);
cudaError_t launch_attn_i8(const SparseI8Launch& a, const CUtensorMap* tm_phik3, const CUtensorMap* tm_v3,
                           cudaStream_t st, int* launches);

// ---- backward (backward.cu): sla2_backward, hard routing, fp32, d / bq / bk <= 64
struct BackwardLaunch {
    int64_t BH, H;
    int N, d, bq, bk, tm, tn;
    int smooth;
    float inv_sqrt_d;
    const float *q, *k, *v, *d_out, *o_s, *o_l, *big_l, *rho;
    const uint8_t* mask;  // [BH][tm][tn]
    float *dq, *dk, *dv, *drho;
    // workspace
    float *mu, *phik, *h, *z, *htot, *ztot, *dh, *dz, *dsr;
};
cudaError_t launch_backward(const BackwardLaunch& a, cudaStream_t st, int* launches);
// phi(K~_j) rows, h_j = phi(K~_j)^T V_j, z_j = colsum phi(K~_j) per key block (mu nullable)
cudaError_t launch_keyblock_linear(const float* k, const float* v, const float* mu, float* phik, float* h, float* z,
                                   int64_t BH, int N, int d, int bk, cudaStream_t st, int* launches);

// ---- stage-1 soft routing (soft.cu): soft_topk + the SoftMask forward, fp32, d / bq / bk <= 64
cudaError_t launch_soft_topk(const float* pc, int rows, int tn, double kappa, double tau, float* values,
                             float* lambdas, int* fail, cudaStream_t st, int* launches);
cudaError_t launch_soft_topk_backward(const float* values, const float* upstream, float* grad, int64_t n,
                                      float inv_tau, cudaStream_t st, int* launches);
struct SoftLaunch {
    int64_t BH, H;
    int N, d, bq, bk, tm, tn;
    float inv_sqrt_d;
    const float *q, *k, *v, *mu, *values, *rho, *h, *z;  // mu nullable (smooth off)
    float *out, *o_s, *o_l, *big_l;                      // o_s / o_l / big_l nullable
};
cudaError_t launch_soft_forward(const SoftLaunch& a, cudaStream_t st, int* launches);

}  // namespace sla2dev
