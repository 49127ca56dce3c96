// sparse_f32.cu -- fp32 SLA2 forward (config 1: fp32, tolerance 1e-4) on CUDA cores.
//
// tcgen05 has no fp32 kind, so the fp32 configuration runs on the FFMA pipe. Same algorithm
// as sparse_bf16.cu, generic in (d <= 128, bq | 256, bk <= 128): one CTA per (query block i,
// bh), each thread owning one row of O (threads-per-row = 256 / bq). Follows
// sla2_forward_blockwise (attention.hpp:484-558): S on K~ = K - mu (block_scores_qk 372-394,
// fp32 path), online softmax with exact rescale (506-523), O += P V (block_product_pv
// 396-415), complement as Htot - Hsel (495-502), epilogue 532-557.
#include <cuda_runtime.h>

#include <cstdint>

#include "expf_glibc.cuh"
#include "kernels.h"

namespace sla2dev {

size_t sparse_f32_smem_bytes(int d, int bq, int bk) {
    const size_t main_ = (size_t)bq * d + (size_t)bk * (d + 1) + 2 * (size_t)bk * d + (size_t)bq * (bk + 1);
    const size_t epi = (size_t)bq * d + (size_t)d * d;  // sQ stays, Hc aliases the key tiles
    const size_t fl = (main_ > epi ? main_ : epi) + d;
    return fl * sizeof(float);
}

template <int TPR>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int TPR>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int TPR>
__global__ void __launch_bounds__(256) sla2_sparse_f32_kernel(SparseLaunch a) {
    extern __shared__ float sm[];
    const int d = a.d, bq = a.bq, bk = a.bk;
    const int i = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int h = (int)(bh % a.H);
    const int tid = threadIdx.x;
    const int r = tid / TPR, q = tid % TPR;
    const bool act = r < bq;  // bq < 8: the row groups past bq only help with the Hsel entries
    const bool dense = a.dense != 0;
    const int nb = dense ? a.tn : (a.kv_cnt ? a.kv_cnt[bh * a.tm + i] : a.kappa);
    const int32_t* idx = a.kv_idx + (bh * a.tm + i) * (int64_t)a.kstride;
    const bool full_row = dense || nb == a.tn;

    float* sQ = sm;                    // [bq][d]
    float* sK = sQ + bq * d;           // [bk][d+1]
    float* sV = sK + bk * (d + 1);     // [bk][d]
    float* sPh = sV + bk * d;          // [bk][d]
    float* sP = sPh + bk * d;          // [bq][bk+1]
    float* sHc = sQ + bq * d;          // epilogue alias [d][d]
    const size_t main_ = (size_t)bq * d + (size_t)bk * (d + 1) + 2 * (size_t)bk * d + (size_t)bq * (bk + 1);
    const size_t epi = (size_t)bq * d + (size_t)d * d;
    float* sZc = sm + (main_ > epi ? main_ : epi);  // [d]

    const float* mu = (a.smooth && a.mu) ? a.mu + bh * d : nullptr;
    const int64_t qrow0 = bh * a.N + (int64_t)i * bq;
    for (int e = tid; e < bq * d; e += 256) sQ[e] = a.q[qrow0 * d + e];

    constexpr int MAXC = 64;  // O columns per thread (d / TPR <= 64)
    float o[MAXC];
    const int nc = (act && q < d) ? (d - q + TPR - 1) / TPR : 0;  // O columns c = q + TPR*u of this thread
    for (int u = 0; u < nc; ++u) o[u] = 0.0f;
    float hs[64];
    const int dd = d * d;
    const int nh = (dd + 255) / 256;
    for (int u = 0; u < nh; ++u) hs[u] = 0.0f;
    float m = -INFINITY, l = 0.0f;
    const int ns = (act && q < bk) ? (bk - q + TPR - 1) / TPR : 0;  // S entries t = q + TPR*v of this thread

    for (int jj = 0; jj < nb; ++jj) {
        const int kb = dense ? jj : idx[jj];
        const int64_t krow0 = bh * a.N + (int64_t)kb * bk;
        __syncthreads();
        for (int e = tid; e < bk * d; e += 256) {
            const int t = e / d, f = e % d;
            const float kv = a.k[krow0 * d + e];
            sK[t * (d + 1) + f] = mu ? kv - mu[f] : kv;
            sV[e] = a.v[krow0 * d + e];
            if (!full_row) sPh[e] = a.phik[krow0 * d + e];
        }
        __syncthreads();
        float s[64];
        float mx = -INFINITY;
        for (int v = 0; v < ns; ++v) {
            const int t = q + TPR * v;
            float acc = 0.0f;
            for (int f = 0; f < d; ++f) acc = fmaf(sQ[r * d + f], sK[t * (d + 1) + f], acc);
            s[v] = acc * a.inv_sqrt_d;
            mx = fmaxf(mx, s[v]);
        }
        mx = group_max<TPR>(mx);
        const float m_new = fmaxf(m, mx);
        const float corr = expf(m - m_new);
        float rs = 0.0f;
        for (int v = 0; v < ns; ++v) {
            const float pv = expf(s[v] - m_new);
            rs += pv;
            sP[r * (bk + 1) + q + TPR * v] = pv;
        }
        rs = group_sum<TPR>(rs);
        l = corr * l + rs;
        m = m_new;
        for (int u = 0; u < nc; ++u) o[u] *= corr;
        __syncthreads();
        for (int u = 0; u < nc; ++u) {
            const int c = q + TPR * u;
            float acc = o[u];
            for (int t = 0; t < bk; ++t) acc = fmaf(sP[r * (bk + 1) + t], sV[t * d + c], acc);
            o[u] = acc;
        }
        if (!full_row) {
            for (int u = 0; u < nh; ++u) {
                const int e = tid + 256 * u;
                if (e < dd) {
                    const int f = e / d, c = e % d;
                    float acc = hs[u];
                    for (int t = 0; t < bk; ++t) acc = fmaf(sPh[t * d + f], sV[t * d + c], acc);
                    hs[u] = acc;
                }
            }
        }
    }
    __syncthreads();

    float alpha = 1.0f;
    if (!full_row) {
        const float x = a.rho[(int64_t)h * a.tm + i];
        float av = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x)));
        alpha = fminf(fmaxf(av, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
        const float* ht = a.htot + bh * (int64_t)dd;
        for (int u = 0; u < nh; ++u) {
            const int e = tid + 256 * u;
            if (e < dd) sHc[e] = ht[e] - hs[u];
        }
        const float* zb = a.zblk + bh * (int64_t)a.tn * d;
        for (int f = tid; f < d; f += 256) {
            float sel = 0.0f;
            for (int jj = 0; jj < nb; ++jj) sel += zb[(int64_t)idx[jj] * d + f];
            sZc[f] = a.ztot[bh * d + f] - sel;
        }
    }
    if (a.h_blocks) {  // SLA2ForwardSaved h_blocks / z_blocks (zero on full rows, attention.hpp:495)
        __syncthreads();
        const int64_t tile = bh * a.tm + i;
        for (int e = tid; e < dd; e += 256) a.h_blocks[tile * dd + e] = full_row ? 0.0f : sHc[e];
        for (int f = tid; f < d; f += 256) a.z_blocks[tile * d + f] = full_row ? 0.0f : sZc[f];
    }
    __syncthreads();
    const int64_t grow = qrow0 + r;
    const float inv_l = 1.0f / l;
    float* out = reinterpret_cast<float*>(a.out) + grow * d;
    if (!full_row) {
        // phi(Q_r) = row softmax over d (attention.hpp:456)
        float qm = -INFINITY;
        for (int f = 0; f < d; ++f) qm = fmaxf(qm, sQ[r * d + f]);
        float qs = 0.0f;
        for (int f = 0; f < d; ++f) qs += expf(sQ[r * d + f] - qm);
        const float qinv = 1.0f / qs;
        float den = 0.0f;
        for (int f = 0; f < d; ++f) den = fmaf(expf(sQ[r * d + f] - qm) * qinv, sZc[f], den);
        for (int u = 0; u < nc; ++u) {
            const int c = q + TPR * u;
            float num = 0.0f;
            for (int f = 0; f < d; ++f) num = fmaf(expf(sQ[r * d + f] - qm) * qinv, sHc[f * d + c], num);
            const float os = o[u] * inv_l;
            const float ol = num / den;
            out[c] = alpha * os + (1.0f - alpha) * ol;
            if (a.o_s) a.o_s[grow * d + c] = os;
            if (a.o_l) a.o_l[grow * d + c] = ol;
        }
    } else {
        for (int u = 0; u < nc; ++u) {
            const int c = q + TPR * u;
            const float os = o[u] * inv_l;
            out[c] = os;
            if (a.o_s) a.o_s[grow * d + c] = os;
            if (a.o_l) a.o_l[grow * d + c] = 0.0f;
        }
    }
    if (act && a.big_l && q == 0) a.big_l[grow] = m + logf(l);
}

cudaError_t launch_sparse_f32(const SparseLaunch& a, cudaStream_t st, int* launches) {
    const size_t smem = sparse_f32_smem_bytes(a.d, a.bq, a.bk);
    dim3 grid(a.tm, (unsigned)(a.B * a.H));
    const int tpr = a.bq >= 8 ? 256 / a.bq : 32;  // bq < 8: 8 row groups, the extra ones idle
#define SLA2_F32_CASE(T)                                                                              \
    case T:                                                                                           \
        cudaFuncSetAttribute(sla2_sparse_f32_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                              \
        sla2_sparse_f32_kernel<T><<<grid, 256, smem, st>>>(a);                                        \
        break;
    switch (tpr) {
        SLA2_F32_CASE(1)
        SLA2_F32_CASE(2)
        SLA2_F32_CASE(4)
        SLA2_F32_CASE(8)
        SLA2_F32_CASE(16)
        SLA2_F32_CASE(32)
        default:
            return cudaErrorInvalidValue;
    }
#undef SLA2_F32_CASE
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
