/*
 * sla2_capi.h -- C ABI of libsla2_b200.so, the B200-native (sm_100a) SLA2 forward pass.
 *
 * This is the drop-in boundary for the reference's hot path, the header-only C++ library in
 * /root/reference/proj/include/sla2. Each entry point below replaces one reference
 * interface (cited); the C++ shim include/sla2_b200/sla2.hpp re-exposes the reference's own
 * names and types (sla2::block_scores, sla2::hard_topk, sla2::sla2_forward_blockwise, ...)
 * on top of these calls, and INTEGRATION.md shows the bindings a maintainer adds.
 *
 * Conventions
 *   - Plain pointers and sizes only. Tensors are contiguous row-major
 *     [B, H, N, d] (q, k, v, out) -- each (b, h) slice is exactly one reference
 *     sla2::Matrix<T> (matrix.hpp:18-23). Per-head router state is [H, d, d] (proj_q,
 *     proj_k, the RouterParams<float> of model.hpp:38,94) and [H, tm] (rho, the MixRatio
 *     logits of model.hpp:39,95), both float32.
 *   - "Device" entry points take device pointers, a caller-owned device workspace
 *     (size from sla2_workspace_size) and a cudaStream_t passed as void*; they never
 *     allocate and are stream-ordered. "_host" entry points take host pointers and do the
 *     copies themselves (the reference's value-semantics call shape).
 *   - Errors: the return code is the reference's exception class (common.hpp:13-29):
 *     SLA2_SHAPE_ERROR <-> sla2::shape_error, SLA2_NUMERIC_ERROR <-> sla2::numeric_error,
 *     SLA2_CONTRACT_ERROR <-> sla2::contract_error; SLA2_CUDA_ERROR for a failed launch /
 *     missing sm_100a device. All validation runs on the host before any launch, like the
 *     reference's validation prologues. sla2_last_error() gives the message (thread-local).
 *   - No CPU fallback exists: without an sm_100a device every compute call returns
 *     SLA2_CUDA_ERROR.
 */
#ifndef SLA2_CAPI_H
#define SLA2_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SLA2_OK = 0,
    SLA2_SHAPE_ERROR = 1,    /* sla2::shape_error    */
    SLA2_NUMERIC_ERROR = 2,  /* sla2::numeric_error  */
    SLA2_CONTRACT_ERROR = 3, /* sla2::contract_error */
    SLA2_CUDA_ERROR = 4
} sla2_status;

typedef enum { SLA2_F32 = 0, SLA2_BF16 = 1 } sla2_dtype;

/* QuantConfig (quant.hpp:15-19): NONE = nullptr, INT8 = {bits 8, qk_product, pv_product}. */
/* SLA2_QUANT_FP8PV is not a reference mode (the reference is INT8-only): the paper's low-bit
 * P/V product in E4M3 on kind::f8f6f4 (P unscaled, V with one scale per head, phi(K~) x 448),
 * bf16 Q K^T, fp32 accumulation; bf16 path, out only; checked within the bf16 tolerance. */
typedef enum { SLA2_QUANT_NONE = 0, SLA2_QUANT_INT8 = 1, SLA2_QUANT_FP8PV = 2 } sla2_quant;

typedef struct {
    int64_t B, H, N, d; /* batch, heads, tokens, head dim. N % bq == N % bk == 0 as the reference
                         * requires (attention.hpp:39-41), except on the bf16 non-QAT path, which
                         * also takes a ragged N (e.g. Wan's 32760 / 75600): the last query / key
                         * block is partial, pooled over its own rows, and keys past N are masked
                         * (the oracle's sla2o_*_ragged extension). tm = ceil(N/bq), tn = ceil(N/bk). */
    int64_t bq, bk;     /* block sizes (AttentionInputs::bq/bk, attention.hpp:27-28) */
    double k_percent;   /* router budget, hard_topk (router.hpp:106-125); in (0, 100] */
    int32_t dtype;      /* sla2_dtype of q, k, v, out */
    int32_t quant;      /* sla2_quant */
    int32_t smooth;     /* smooth_k on (the reference default `smooth = true`) */
    int32_t exact_mu;   /* 1: K column mean in the reference's serial order (bit-exact mask);
                           0: tree-reduced mean (faster, mask may differ at fp32 ties) */
    float tau;          /* RouterParams::tau, validated > 0 (router.hpp:32); unused by hard top-k */
    int32_t reserved[3];
} sla2_fwd_params;

/* Optional saved state (SLA2ForwardSaved, attention.hpp:345-358), fp32, device; every member
 * may be NULL. o_l requires o_s. The routing/flags/block sizes of the reference struct are the
 * caller's own inputs (mask_out / kv_idx_out, p). */
typedef struct {
    float* o_s;      /* [B,H,N,d] sparse-branch output O_s */
    float* o_l;      /* [B,H,N,d] linear-branch output O_l (rows of full mask rows = 0) */
    float* big_l;    /* [B,H,N] logsumexp L = m + log l */
    float* h_blocks; /* [B,H,tm,d,d] per query block complement H_i = sum over unselected j of
                      * h_j = phi(K~_j)^T V_j (attention.hpp:495-502; formed as total minus
                      * selected, tolerance-level; zero for full rows) */
    float* z_blocks; /* [B,H,tm,d] complement Z_i = sum over unselected j of colsum phi(K~_j) */
    float* q_phi;    /* [B,H,N,d] phi(Q) = row_softmax(Q) (attention.hpp:456), exact arithmetic */
    float* k_phi;    /* [B,H,N,d] phi(K~) = row_softmax(K - colmean K) (457), exact arithmetic */
    float* qat_s_first; /* QAT only, parity hook: [B,H,tm,bq,bk] the dequantized scores S of each
                      * query block's first kept key block (block_scores_qk, 372-394) */
} sla2_fwd_saved;

/* Fills p with the reference defaults for one (B, H, N, d) problem: bq = 128, bk = 64
 * (PAPER.md:476), k_percent = 3, bf16, no quant, smooth = 1, exact_mu = 1, tau = 0.1. */
void sla2_default_params(sla2_fwd_params* p, int64_t B, int64_t H, int64_t N, int64_t d);

/* topk_budget (router.hpp:36-40): kappa = min(tn, max(1, llround(k% / 100 * tn))). */
int64_t sla2_topk_budget(double k_percent, int64_t tn);

/* Validates p exactly as the reference's prologues would (router.hpp:27-33,90-94,108-110;
 * attention.hpp:36-43,427-447; matrix.hpp:175-179) plus this build's kernel limits. */
sla2_status sla2_check_params(const sla2_fwd_params* p);

/* Bytes of device workspace sla2_forward / sla2_router / sla2_sparse_fwd need for p. */
size_t sla2_workspace_size(const sla2_fwd_params* p);

/*
 * Full forward, replacing Tape::sla2_attention's composition (tape.hpp:263-272):
 *   K~ = smooth_k(K)                          (quant.hpp:88-96)
 *   pc = block_scores(Q, K~, router, bq, bk)  (router.hpp:87-102)
 *   M  = hard_topk(pc, k_percent)             (router.hpp:106-125)
 *   out = sla2_forward_blockwise(Q, K, V, M, rho, quant, smooth)  (attention.hpp:423-560)
 * mask_out [B,H,tm,tn] u8 (BlockMask::bits) and kv_idx_out [B,H,tm,kappa] int32 (each
 * row's kept key blocks, ascending) are optional (NULL = not written).
 */
sla2_status sla2_forward(const sla2_fwd_params* p, const void* q, const void* k, const void* v,
                         const float* proj_q, const float* proj_k, const float* rho, void* out,
                         uint8_t* mask_out, int32_t* kv_idx_out, const sla2_fwd_saved* saved,
                         void* workspace, size_t workspace_bytes, void* stream);

/*
 * Router only: smooth_k + block_scores + hard_topk, bit-exact with the reference.
 * pc_out [B,H,tm,tn] fp32 (the row-softmaxed block scores) may be NULL.
 */
sla2_status sla2_router(const sla2_fwd_params* p, const void* q, const void* k, const float* proj_q,
                        const float* proj_k, float* pc_out, uint8_t* mask_out, int32_t* kv_idx_out,
                        void* workspace, size_t workspace_bytes, void* stream);

/*
 * smooth_k (quant.hpp:88-96) on device: mean_out [B,H,d] fp32 and, if ktilde_out is not NULL,
 * K~ = K - mean as fp32 [B,H,N,d].
 */
sla2_status sla2_smooth_k(const sla2_fwd_params* p, const void* k, float* mean_out, float* ktilde_out,
                          void* stream);

/*
 * hard_topk (router.hpp:106-125) on a caller-given score matrix pc [B,H,tm,tn] fp32: per row
 * the kappa largest entries, ties to the lowest column, as mask bits and ascending index lists.
 */
sla2_status sla2_hard_topk(const sla2_fwd_params* p, const float* pc, uint8_t* mask_out,
                           int32_t* kv_idx_out, void* stream);

/*
 * The linear branch's key-side precompute (attention.hpp:456-475): K~ = K - colmean(K) (p->smooth),
 * phi(K~) = row_softmax(K~) and, per key block j, z_j = colsum phi(K~_j), with the head totals
 * H = sum_j phi(K~_j)^T V_j (d x d) and Z = sum_j z_j that the forward's complements are formed
 * from ("total minus selected", attention.hpp:495-502). Outputs (device, fp32, each nullable):
 * k_phi_out [B,H,N,d] (exact row softmax), z_blocks_out [B,H,tn,d], h_total_out [B,H,d,d],
 * z_total_out [B,H,d]. On the bf16 path z_j and H are accumulated from the bf16-rounded phi(K~)
 * the sparse kernel reads (tolerance-level). The per-key-block h_j matrices are not
 * materialized (the forward needs only H and the selected sums). Workspace:
 * sla2_workspace_size(p).
 */
sla2_status sla2_linear_precompute(const sla2_fwd_params* p, const void* k, const void* v, float* k_phi_out,
                                   float* z_blocks_out, float* h_total_out, float* z_total_out, void* workspace,
                                   size_t workspace_bytes, void* stream);

/*
 * The QAT operand quantization (quantize, quant.hpp:31-50, on the blocks block_scores_qk and
 * block_product_pv quantize, attention.hpp:379-380,401): per query block Q_i (bq x d), per key
 * block K~_j = K_j - colmean(K) (bk x d, when p->smooth) and V_j (bk x d), the absmax/127 scale
 * and the round-half-away codes in [-127, 127], bit-exact with the reference. q/k/v bf16
 * [B,H,N,d]; codes int8 [B,H,N,d] (row-major, each block's rows contiguous); scales fp32
 * q [B,H,tm], k and v [B,H,tn]. p: dtype bf16, quant int8. Workspace: sla2_workspace_size(p).
 * This is the precompute sla2_forward runs before the kind::i8 kernel (exposed for parity).
 */
sla2_status sla2_quantize(const sla2_fwd_params* p, const void* q, const void* k, const void* v, int8_t* q_codes,
                          float* q_scales, int8_t* k_codes, float* k_scales, int8_t* v_codes, float* v_scales,
                          void* workspace, size_t workspace_bytes, void* stream);

/*
 * sla2_forward_blockwise (attention.hpp:423-560) with a caller-given BlockMask (device
 * [B,H,tm,tn] u8, any number of kept blocks per row, e.g. BlockMask::ones). A row that keeps
 * no block returns SLA2_SHAPE_ERROR like the reference (attention.hpp:442-447); checking it
 * costs one device->host read, so this entry point synchronizes `stream` once.
 * p->k_percent is not used.
 */
sla2_status sla2_sparse_fwd(const sla2_fwd_params* p, const void* q, const void* k, const void* v,
                            const float* rho, const uint8_t* mask, void* out, const sla2_fwd_saved* saved,
                            void* workspace, size_t workspace_bytes, void* stream);

/*
 * Dense softmax attention softmax(QK^T / sqrt d) V (full_attention, attention.hpp:71-75): the
 * same tcgen05 kernel visiting every key block -- the "dense sm_100a attention of the same
 * build" the north-star compares against. bf16 only.
 */
sla2_status sla2_dense_fwd(const sla2_fwd_params* p, const void* q, const void* k, const void* v, void* out,
                           void* workspace, size_t workspace_bytes, void* stream);

/*
 * SLA2 backward with hard routing (sla2_backward, attention.hpp:610-809; the stage-2 / QAT
 * fine-tuning path). Full precision whatever the forward was (the QAT contract):
 * fp32 q, k, v, d_out [B,H,N,d]; the routing mask [B,H,tm,tn] (u8, every row keeps a block);
 * rho [H,tm]; the forward's saved o_s, o_l [B,H,N,d] and big_l [B,H,N] (sla2_forward with
 * `saved`). Writes dq, dk, dv [B,H,N,d] and drho [B,H,tm] (per (b,h); sum over b for the
 * shared per-head logits). params: dtype SLA2_F32, d <= 128, bk <= 64, bq <= 64 or a multiple
 * of 64 (<= 128 when d > 64: the Wan2.1 block shape d = 128, bq = 128, bk = 64), N divisible,
 * tm <= 1024; smooth as in the forward. SoftMask routing (stage 1) is not on this path.
 * The workspace is sla2_backward_workspace_size(p) bytes.
 */
size_t sla2_backward_workspace_size(const sla2_fwd_params* p);
sla2_status sla2_backward(const sla2_fwd_params* p, const void* q, const void* k, const void* v, const float* rho,
                          const uint8_t* mask, const float* o_s, const float* o_l, const float* big_l,
                          const void* d_out, void* dq, void* dk, void* dv, float* drho, void* workspace,
                          size_t workspace_bytes, void* stream);

/*
 * Stage-1 soft routing (the router-training path, training.hpp:186-201).
 *
 * sla2_soft_topk replaces soft_topk (router.hpp:126-190): per row of pc [B,H,tm,tn] fp32, the
 * shift lambda_i found by bisection (<= 200 halvings, |row sum - kappa| <= 1e-6, in double) with
 * values_ij = clamp(sigma(pc_ij / tau + lambda_i), DBL_MIN, 1 - eps/2) cast to fp32; kappa =
 * sla2_topk_budget(p->k_percent, tn), tau = p->tau. Writes values [B,H,tm,tn] and lambdas
 * [B,H,tm]. A row that does not converge returns SLA2_NUMERIC_ERROR like the reference's throw
 * (the check is one device->host read: this call synchronizes `stream`).
 *
 * sla2_forward_soft replaces sla2_forward_blockwise with Routing = SoftMask (attention.hpp:
 * 484-558): every key block j of query block i feeds the sparse branch with weight w_ij =
 * values_ij and the linear branch with 1 - w_ij; there are no full rows, so out = alpha O_s +
 * (1 - alpha) O_l. fp32 q, k, v, out [B,H,N,d], values [B,H,tm,tn], rho [H,tm]; saved as in
 * sla2_forward. params: dtype SLA2_F32, no quant, d, bq, bk <= 64, N divisible; smooth as in
 * the reference. Workspace: sla2_forward_soft_workspace_size(p) bytes.
 */
sla2_status sla2_soft_topk(const sla2_fwd_params* p, const float* pc, float* values, float* lambdas, void* stream);
/* soft_topk_backward (router.hpp:197-212): the frozen-lambda gradient grad = upstream * v *
 * (1 - v) / tau elementwise over [B,H,tm,tn] (values from sla2_soft_topk, tau = p->tau). */
sla2_status sla2_soft_topk_backward(const sla2_fwd_params* p, const float* values, const float* upstream,
                                    float* grad, void* stream);
size_t sla2_forward_soft_workspace_size(const sla2_fwd_params* p);
sla2_status sla2_forward_soft(const sla2_fwd_params* p, const void* q, const void* k, const void* v, const float* rho,
                              const float* values, void* out, const sla2_fwd_saved* saved, void* workspace,
                              size_t workspace_bytes, void* stream);

/*
 * Host-buffer forward: the reference's call shape (inputs and outputs in host memory).
 * Copies q/k/v/proj/rho host->device, runs sla2_forward on an internal stream with an
 * internally cached workspace, copies out (and the optional mask) back, synchronizes.
 * Pipelined per (b, h): the H2D of head c+1 and the D2H of head c-1 overlap the compute of
 * head c on three streams (pinned host buffers make the copies asynchronous). Results are
 * identical to one sla2_forward over all heads.
 */
sla2_status sla2_forward_host(const sla2_fwd_params* p, const void* q, const void* k, const void* v,
                              const float* proj_q, const float* proj_k, const float* rho, void* out,
                              uint8_t* mask_out);

/* Message of the last error on this thread ("" if none). */
const char* sla2_last_error(void);

/* Number of kernel launches the last sla2_* call on this thread enqueued (bench evidence). */
int32_t sla2_last_launch_count(void);

/* Stage timing (off by default). When enabled, sla2_forward records CUDA events on its
 * stream around its stages; sla2_last_stage_ms waits for the last call's events and writes
 * up to n durations in ms: [0] router (smooth_k + block_scores + hard_topk), [1] linear
 * precompute (phi(K~), z, Htot), [2] sparse+linear+blend kernel, [3] whole call; then the
 * timeline in ms since the call started (-1 when the path did not pass the point): [4] mu
 * ready, [5] query side done, [6] key prep done, [7] router back half done, [8] linear
 * precompute done. The router and the linear precompute overlap on two streams, so [1] is
 * only the wait for the latter. Returns the number written (<= 9). */
void sla2_enable_stage_timing(int32_t enable);
int32_t sla2_last_stage_ms(float* out, int32_t n);

/* "sla2_b200 <version> sm_100a" */
const char* sla2_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SLA2_CAPI_H */
