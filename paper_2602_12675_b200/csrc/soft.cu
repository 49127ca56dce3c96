// soft.cu -- stage-1 (soft routing) SLA2 forward on sm_100a, fp32 CUDA cores.
//
// Replaces, on the SoftMask path of Tape-level training stage 1:
//   soft_topk (router.hpp:126-190): per row, bisection (<= 200 halvings, |sum - kappa| <= 1e-6) for
//     lambda_i with values_ij = clamp(sigma(pc_ij / tau + lambda_i), DBL_MIN, 1 - eps/2), in double;
//   sla2_forward_blockwise with Routing = SoftMask (attention.hpp:484-558): every key block j of
//     query block i contributes w_ij to the sparse branch (l = rescale l + w rs, o = o rescale +
//     w P V) and cw_ij = 1 - w_ij to the linear branch (H_i += cw h_j, Z_i += cw z_j); there are
//     no full rows, so out = alpha O_s + (1 - alpha) O_l.
// The soft mask visits every block (stage 1 trains the router densely); this first version is a
// per-query-block CUDA-core kernel for d, bq, bk <= 64, like the backward. phi(K~), h_j and z_j
// come from backward.cu's bwd_keyblock_kernel (launch_keyblock_linear).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "kernels.h"

namespace sla2dev {
namespace sf {
constexpr int MAXD = 64, MAXB = 64;
}

// one warp per row; the row sum in double as the reference (lanes own columns j = lane + 32 u)
__global__ void soft_topk_kernel(const float* __restrict__ pc, int rows, int tn, double kappa, double tau,
                                 float* __restrict__ values, float* __restrict__ lambdas, int* __restrict__ fail) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* p = pc + (int64_t)row * tn;
    double mn = 1e300, mx = -1e300;
    for (int j = lane; j < tn; j += 32) {
        mn = fmin(mn, (double)p[j]);
        mx = fmax(mx, (double)p[j]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    double lo = -mx / tau - 40.0, hi = -mn / tau + 40.0, lam = 0.0, resid = 0.0;
    bool converged = false;
    for (int iter = 0; iter < 200; ++iter) {
        lam = 0.5 * (lo + hi);
        double s = 0.0;
        for (int j = lane; j < tn; j += 32) s += 1.0 / (1.0 + exp(-((double)p[j] / tau + lam)));
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        resid = s - kappa;
        if (fabs(resid) <= 1e-6) {
            converged = true;
            break;
        }
        if (resid > 0.0) hi = lam;
        else lo = lam;
    }
    if (!converged && lane == 0) atomicExch(fail, 1);  // the reference throws numeric_error
    if (lane == 0) lambdas[row] = (float)lam;
    for (int j = lane; j < tn; j += 32) {
        double v = 1.0 / (1.0 + exp(-((double)p[j] / tau + lam)));
        v = fmin(fmax(v, DBL_MIN), 1.0 - DBL_EPSILON / 2);
        values[(int64_t)row * tn + j] = (float)v;
    }
}

// soft_topk_backward (router.hpp:197-212): frozen-lambda diagonal Jacobian,
// grad = upstream * v * (1 - v) * (1 / tau), left to right as the reference
__global__ void soft_topk_backward_kernel(const float* __restrict__ values, const float* __restrict__ upstream,
                                          float* __restrict__ grad, int64_t n, float inv_tau) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const float v = values[e];
        grad[e] = __fmul_rn(__fmul_rn(__fmul_rn(upstream[e], v), __fsub_rn(1.0f, v)), inv_tau);
    }
}

// per (bh, query block): the weighted sparse and linear branches over every key block
__global__ void __launch_bounds__(256) soft_forward_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ mu, const float* __restrict__ values, const float* __restrict__ rho,
    const float* __restrict__ h, const float* __restrict__ z, float* __restrict__ out, float* __restrict__ o_s,
    float* __restrict__ o_l, float* __restrict__ big_l, int N, int d, int bq, int bk, int tm, int tn, int H,
    float inv_sqrt_d) {
    extern __shared__ float sm[];
    const int ld = sf::MAXD + 1, pl = sf::MAXB + 1;
    float* sq = sm;                   // [bq][ld] Q_i
    float* sk = sq + sf::MAXB * ld;   // [bk][ld] K~_j
    float* sv = sk + sf::MAXB * ld;   // [bk][ld] V_j
    float* sp = sv + sf::MAXB * ld;   // [bq][pl] S, then P
    float* so = sp + sf::MAXB * pl;   // [bq][ld] o accumulator
    float* shi = so + sf::MAXB * ld;  // [d][ld]  H_i
    __shared__ float szi[sf::MAXD], smr[sf::MAXB], slr[sf::MAXB], sresc[sf::MAXB];
    const int i = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int hh = (int)(bh % H);
    const int64_t r0 = bh * N + (int64_t)i * bq;
    for (int e = threadIdx.x; e < bq * d; e += blockDim.x) {
        const int r = e / d, c = e % d;
        sq[r * ld + c] = q[(r0 + r) * d + c];
        so[r * ld + c] = 0.0f;
    }
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) shi[(e / d) * ld + e % d] = 0.0f;
    for (int f = threadIdx.x; f < d; f += blockDim.x) szi[f] = 0.0f;
    for (int r = threadIdx.x; r < bq; r += blockDim.x) {
        smr[r] = -INFINITY;
        slr[r] = 0.0f;
    }
    const float* wrow = values + (bh * tm + i) * (int64_t)tn;
    for (int j = 0; j < tn; ++j) {
        const float w = wrow[j], cw = 1.0f - w;
        __syncthreads();
        if (cw > 0.0f) {  // attention.hpp:495-502
            const float* hj = h + (bh * tn + j) * (int64_t)d * d;
            for (int e = threadIdx.x; e < d * d; e += blockDim.x) shi[(e / d) * ld + e % d] += cw * hj[e];
            for (int f = threadIdx.x; f < d; f += blockDim.x) szi[f] += cw * z[(bh * tn + j) * d + f];
        }
        if (w <= 0.0f) continue;
        const int64_t c0 = bh * N + (int64_t)j * bk;
        for (int e = threadIdx.x; e < bk * d; e += blockDim.x) {
            const int t = e / d, c = e % d;
            sk[t * ld + c] = k[(c0 + t) * d + c] - (mu ? mu[bh * d + c] : 0.0f);
            sv[t * ld + c] = v[(c0 + t) * d + c];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < bq * bk; e += blockDim.x) {  // S = Q K~^T / sqrt(d)
            const int r = e / bk, t = e % bk;
            float acc = 0.0f;
            for (int f = 0; f < d; ++f) acc += sq[r * ld + f] * sk[t * ld + f];
            sp[r * pl + t] = acc * inv_sqrt_d;
        }
        __syncthreads();
        for (int r = threadIdx.x; r < bq; r += blockDim.x) {  // online softmax (attention.hpp:506-521)
            float mx = sp[r * pl];
            for (int t = 1; t < bk; ++t) mx = fmaxf(mx, sp[r * pl + t]);
            const float m_new = fmaxf(smr[r], mx);
            const float rescale = expf(smr[r] - m_new);
            float rs = 0.0f;
            for (int t = 0; t < bk; ++t) {
                const float pt = expf(sp[r * pl + t] - m_new);
                sp[r * pl + t] = pt;
                rs += pt;
            }
            slr[r] = rescale * slr[r] + w * rs;
            smr[r] = m_new;
            sresc[r] = rescale;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < bq * d; e += blockDim.x) {  // o = o rescale + w (P V)
            const int r = e / d, c = e % d;
            float acc = 0.0f;
            for (int t = 0; t < bk; ++t) acc += sp[r * pl + t] * sv[t * ld + c];
            so[r * ld + c] = so[r * ld + c] * sresc[r] + w * acc;
        }
    }
    __syncthreads();
    // epilogue (attention.hpp:532-557): no full rows on the soft path
    float a = 1.0f / (1.0f + expf(-rho[(int64_t)hh * tm + i]));
    a = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < bq; r += 8) {  // warp per row: phi(Q)_r, den, num
        const int64_t g = r0 + r;
        float qv[2], mx = -INFINITY;
        for (int u = 0; u < 2; ++u) {
            const int f = lane + 32 * u;
            qv[u] = f < d ? sq[r * ld + f] : -INFINITY;
            mx = fmaxf(mx, qv[u]);
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float ph[2], s = 0.0f;
        for (int u = 0; u < 2; ++u) {
            ph[u] = lane + 32 * u < d ? expf(qv[u] - mx) : 0.0f;
            s += ph[u];
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        float den = 0.0f;
        for (int u = 0; u < 2; ++u) {
            ph[u] /= s;
            if (lane + 32 * u < d) den += ph[u] * szi[lane + 32 * u];
        }
        for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
        const float inv_l = 1.0f / slr[r];
        if (lane == 0 && big_l) big_l[g] = smr[r] + logf(slr[r]);
        for (int u = 0; u < 2; ++u) {
            const int c = lane + 32 * u;
            float num = 0.0f;
            for (int f = 0; f < d; ++f) num += __shfl_sync(0xffffffffu, ph[f >> 5], f & 31) * shi[f * ld + (c < d ? c : 0)];
            if (c < d) {
                const float os = so[r * ld + c] * inv_l, ol = num / den;
                if (o_s) o_s[g * d + c] = os;
                if (o_l) o_l[g * d + c] = ol;
                out[g * d + c] = a * os + (1.0f - a) * ol;
            }
        }
    }
}

size_t soft_forward_smem() {
    const int ld = sf::MAXD + 1, pl = sf::MAXB + 1;
    return sizeof(float) * (4 * sf::MAXB * ld + sf::MAXB * pl + sf::MAXD * ld);
}

cudaError_t launch_soft_topk(const float* pc, int rows, int tn, double kappa, double tau, float* values,
                             float* lambdas, int* fail, cudaStream_t st, int* launches) {
    soft_topk_kernel<<<(rows + 7) / 8, 256, 0, st>>>(pc, rows, tn, kappa, tau, values, lambdas, fail);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_soft_topk_backward(const float* values, const float* upstream, float* grad, int64_t n,
                                      float inv_tau, cudaStream_t st, int* launches) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    soft_topk_backward_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(values, upstream, grad, n, inv_tau);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_soft_forward(const SoftLaunch& a, cudaStream_t st, int* launches) {
    if (a.d > sf::MAXD || a.bq > sf::MAXB || a.bk > sf::MAXB) return cudaErrorInvalidValue;
    ensure_smem_attr((const void*)soft_forward_kernel, (int)((int)soft_forward_smem()));
    soft_forward_kernel<<<dim3(a.tm, (unsigned)a.BH), 256, soft_forward_smem(), st>>>(
        a.q, a.k, a.v, a.mu, a.values, a.rho, a.h, a.z, a.out, a.o_s, a.o_l, a.big_l, a.N, a.d, a.bq, a.bk, a.tm,
        a.tn, (int)a.H, a.inv_sqrt_d);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sla2dev
