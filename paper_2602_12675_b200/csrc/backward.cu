// backward.cu -- SLA2 backward with hard routing (stage-2 / QAT fine-tuning), fp32, on sm_100a.
//
// Replaces sla2_backward (attention.hpp:610-809) on the BlockMask path; the QAT contract
// (attention.hpp:735-737) makes it full precision whatever the forward was. Inputs:
// q, k, v, d_out [BH][N][d] fp32, the routing mask [BH][tm][tn], rho [H][tm] and the forward's
// saved O_s, O_l [BH][N][d] and L [BH][N]. Outputs dq, dk, dv [BH][N][d] and drho [BH][tm].
// Everything the reference keeps in SLA2ForwardSaved besides O_s, O_l, L (phi(Q), phi(K~),
// H_i, Z_i) is recomputed here.
//
// Kernels (fp32 CUDA cores, templated on the feature width MD = 64 or 128 so d <= 128; bk <= 64;
// bq <= 64 or a multiple of 64 -- the flash-style kernel takes a query block 64 rows at a time):
//   bwd_keyblock_kernel   phi(K~_j) rows, h_j = phi(K~_j)^T V_j, z_j      (attention.hpp:459-475)
//   bwd_total_kernel      Htot = sum_j h_j, Ztot = sum_j z_j (complement = total - selected)
//   bwd_qblock_kernel     d_os, d_ol, drho, rowsum(d_os o O_s), rowsum(d_ol o O_l); dH_i, dZ_i;
//                         the linear branch's dq through phi's row-softmax Jacobian   (637-690)
//   bwd_sparse_kernel     flash-style recompute of S, P = exp(S - L) per kept block: dq (owned),
//                         dK~ and dV (atomic over query blocks)                          (713-760)
//   bwd_keylin_kernel     dh_tot_j, dz_tot_j over the query blocks that did not keep j; dphi(K~),
//                         its row-softmax Jacobian into dK~, dV_j += phi(K~_j) dh_tot_j  (761-789)
//   bwd_smooth_kernel     dK = dK~ - colmean(dK~)  (smooth_k_backward, quant.hpp:99-107)
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace sla2dev {
namespace bw {
constexpr int MAXB = 64, THREADS = 256;  // key-block rows, query sub-block rows; CTA size
}

// ---------------------------------------------------------------- phi(K~), h_j, z_j
template <int MD>
__global__ void __launch_bounds__(256) bwd_keyblock_kernel(const float* __restrict__ k, const float* __restrict__ v,
                                                           const float* __restrict__ mu, float* __restrict__ phik,
                                                           float* __restrict__ h, float* __restrict__ z, int N, int d,
                                                           int bk) {
    constexpr int NU = MD / 32;
    extern __shared__ float kbsm[];
    float(*sp)[MD + 1] = reinterpret_cast<float(*)[MD + 1]>(kbsm);  // [bk][MD + 1] phi(K~_j)
    float(*sv)[MD + 1] = sp + bw::MAXB;                             // [bk][MD + 1] V_j
    const int j = blockIdx.x, tn = N / bk;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = bh * N + (int64_t)j * bk;
    for (int t = warp; t < bk; t += 8) {  // one warp per key row: row softmax over d (matrix.hpp:138-155)
        float x[NU], mx = -INFINITY;
        for (int u = 0; u < NU; ++u) {
            const int f = lane + 32 * u;
            x[u] = f < d ? k[(row0 + t) * d + f] - (mu ? mu[bh * d + f] : 0.0f) : -INFINITY;
            mx = fmaxf(mx, x[u]);
            if (f < d) sv[t][f] = v[(row0 + t) * d + f];
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float s = 0.0f;
        for (int u = 0; u < NU; ++u) {
            x[u] = lane + 32 * u < d ? expf(x[u] - mx) : 0.0f;
            s += x[u];
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float inv = 1.0f / s;
        for (int u = 0; u < NU; ++u) {
            const int f = lane + 32 * u;
            if (f < d) {
                sp[t][f] = x[u] * inv;
                phik[(row0 + t) * d + f] = x[u] * inv;
            }
        }
    }
    __syncthreads();
    float* hj = h + (bh * tn + j) * (int64_t)d * d;
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int f = e / d, c = e % d;
        float acc = 0.0f;
        for (int t = 0; t < bk; ++t) acc += sp[t][f] * sv[t][c];
        hj[e] = acc;
    }
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
        float acc = 0.0f;
        for (int t = 0; t < bk; ++t) acc += sp[t][f];
        z[(bh * tn + j) * d + f] = acc;
    }
}
template <int MD>
constexpr size_t bwd_keyblock_smem() { return sizeof(float) * 2 * bw::MAXB * (MD + 1); }

__global__ void bwd_total_kernel(const float* __restrict__ h, const float* __restrict__ z, float* __restrict__ htot,
                                 float* __restrict__ ztot, int tn, int d) {
    const int64_t bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < d * d) {
        float acc = 0.0f;
        for (int j = 0; j < tn; ++j) acc += h[(bh * tn + j) * (int64_t)d * d + e];
        htot[bh * d * d + e] = acc;
    }
    if (e < d) {
        float acc = 0.0f;
        for (int j = 0; j < tn; ++j) acc += z[(bh * tn + j) * d + e];
        ztot[bh * d + e] = acc;
    }
}

// ---------------------------------------------------------------- per query block: linear branch
template <int MD>
constexpr size_t bwd_qblock_smem_base() { return sizeof(float) * (MD * (MD + 1) + MD); }
// bytes for a query block of bq rows: Hc, two [bq][MD + 1] row tiles, Zc and the bq row sums
template <int MD>
size_t bwd_qblock_smem(int bq) { return bwd_qblock_smem_base<MD>() + sizeof(float) * (size_t)bq * (2 * (MD + 1) + 1); }

template <int MD>
__global__ void __launch_bounds__(256) bwd_qblock_kernel(
    const float* __restrict__ q, const float* __restrict__ d_out, const float* __restrict__ o_s,
    const float* __restrict__ o_l, const uint8_t* __restrict__ mask, const float* __restrict__ rho,
    const float* __restrict__ h, const float* __restrict__ z, const float* __restrict__ htot,
    const float* __restrict__ ztot, float* __restrict__ dq, float* __restrict__ dsr, float* __restrict__ dh,
    float* __restrict__ dz, float* __restrict__ drho, int N, int d, int bq, int tm, int tn, int H) {
    constexpr int NU = MD / 32;
    extern __shared__ float qsm[];
    float(*shc)[MD + 1] = reinterpret_cast<float(*)[MD + 1]>(qsm);  // [MD] Hc_i = Htot - sum_kept h_j
    float(*sa)[MD + 1] = shc + MD;                                  // [bq] phi(Q)_r / den_r
    float(*sdl)[MD + 1] = sa + bq;                                  // [bq] d_ol rows
    float* szc = reinterpret_cast<float*>(sdl + bq);                // [MD]
    float* sdrl = szc + MD;                                         // [bq] rowsum(d_ol o O_l)
    __shared__ float sred[8];
    __shared__ int sfull;
    const int i = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int h_ = (int)(bh % H);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* mrow = mask + (bh * tm + i) * (int64_t)tn;
    if (threadIdx.x == 0) sfull = 1;
    __syncthreads();
    for (int j = threadIdx.x; j < tn; j += blockDim.x)
        if (!mrow[j]) sfull = 0;
    __syncthreads();
    const bool full = sfull != 0;
    // alpha = sigmoid(rho_i) clamped (attention.hpp:17-22); forced to 1 on full rows (639)
    float av = 1.0f / (1.0f + expf(-rho[(int64_t)h_ * tm + i]));
    av = fminf(fmaxf(av, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
    const float a = full ? 1.0f : av;
    if (!full) {
        const float* hb = h + bh * (int64_t)tn * d * d;
        for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
            float acc = htot[bh * d * d + e];
            for (int j = 0; j < tn; ++j)
                if (mrow[j]) acc -= hb[(int64_t)j * d * d + e];
            shc[e / d][e % d] = acc;
        }
        for (int f = threadIdx.x; f < d; f += blockDim.x) {
            float acc = ztot[bh * d + f];
            for (int j = 0; j < tn; ++j)
                if (mrow[j]) acc -= z[(bh * tn + j) * d + f];
            szc[f] = acc;
        }
    }
    __syncthreads();
    float dalpha = 0.0f;
    for (int r = warp; r < bq; r += 8) {  // one warp per row; lane owns features lane, lane + 32
        const int64_t g = bh * N + (int64_t)i * bq + r;
        float dout[NU], os[NU], ol[NU], qv[NU];
        float srs = 0.0f, srl = 0.0f;
        for (int u = 0; u < NU; ++u) {
            const int c = lane + 32 * u;
            const bool ok = c < d;
            dout[u] = ok ? d_out[g * d + c] : 0.0f;
            os[u] = ok ? o_s[g * d + c] : 0.0f;
            ol[u] = ok ? o_l[g * d + c] : 0.0f;
            qv[u] = ok ? q[g * d + c] : -INFINITY;
            dalpha += dout[u] * (os[u] - ol[u]);
            srs += (a * dout[u]) * os[u];
            srl += ((1.0f - a) * dout[u]) * ol[u];
            if (ok) sdl[r][c] = (1.0f - a) * dout[u];
        }
        for (int o = 16; o > 0; o >>= 1) {
            srs += __shfl_xor_sync(0xffffffffu, srs, o);
            srl += __shfl_xor_sync(0xffffffffu, srl, o);
        }
        if (lane == 0) {
            dsr[g] = srs;
            sdrl[r] = srl;
        }
        float dql[NU];
        for (int u = 0; u < NU; ++u) dql[u] = 0.0f;
        if (!full) {
            // phi(Q)_r (row softmax), den_r = phi(Q)_r . Zc
            float mx = qv[0];
            for (int u = 1; u < NU; ++u) mx = fmaxf(mx, qv[u]);
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float e[NU], s = 0.0f;
            for (int u = 0; u < NU; ++u) {
                e[u] = lane + 32 * u < d ? expf(qv[u] - mx) : 0.0f;
                s += e[u];
            }
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            float ph[NU], den = 0.0f;
            for (int u = 0; u < NU; ++u) {
                ph[u] = e[u] / s;
                den += lane + 32 * u < d ? ph[u] * szc[lane + 32 * u] : 0.0f;
            }
            for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
            const float inv_den = 1.0f / den;
            __syncwarp();
            // dphi(Q)_r[f] = (sum_c d_ol[c] Hc[f][c] - d_row_l Zc[f]) / den   (attention.hpp:682-687)
            float dph[NU], dot = 0.0f;
            for (int u = 0; u < NU; ++u) {
                const int f = lane + 32 * u;
                float acc = 0.0f;
                if (f < d)
                    for (int c = 0; c < d; ++c) acc += sdl[r][c] * shc[f][c];
                dph[u] = f < d ? (acc - srl * szc[f]) * inv_den : 0.0f;
                dot += dph[u] * ph[u];
                if (f < d) sa[r][f] = ph[u] * inv_den;
            }
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            // row_softmax_backward (matrix.hpp:160-169)
            for (int u = 0; u < NU; ++u) dql[u] = ph[u] * (dph[u] - dot);
        }
        for (int u = 0; u < NU; ++u)
            if (lane + 32 * u < d) dq[g * d + lane + 32 * u] = dql[u];
    }
    for (int o = 16; o > 0; o >>= 1) dalpha += __shfl_xor_sync(0xffffffffu, dalpha, o);
    if (lane == 0) sred[warp] = dalpha;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.0f;
        for (int w = 0; w < 8; ++w) t += sred[w];
        drho[bh * tm + i] = full ? 0.0f : t * av * (1.0f - av);  // attention.hpp:648-651
    }
    // dH_i[f][c] = sum_r (phi(Q)_r[f] / den_r) d_ol[r][c], dZ_i[f] = -sum_r (...) d_row_l[r]
    float* dhi = dh + (bh * tm + i) * (int64_t)d * d;
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int f = e / d, c = e % d;
        float acc = 0.0f;
        if (!full)
            for (int r = 0; r < bq; ++r) acc += sa[r][f] * sdl[r][c];
        dhi[e] = acc;
    }
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
        float acc = 0.0f;
        if (!full)
            for (int r = 0; r < bq; ++r) acc -= sa[r][f] * sdrl[r];
        dz[(bh * tm + i) * d + f] = acc;
    }
}

// ---------------------------------------------------------------- sparse branch (flash-style)
// One CTA per (query block i, 64-row sub-block): the rows of a query block are independent in
// the recompute (their own L, dsr, dq), and dK~ / dV are atomic over query blocks anyway.
template <int MD>
__global__ void __launch_bounds__(256) bwd_sparse_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ mu, const float* __restrict__ d_out, const float* __restrict__ big_l,
    const float* __restrict__ dsr, const uint8_t* __restrict__ mask, const float* __restrict__ rho,
    float* __restrict__ dq, float* __restrict__ dkt, float* __restrict__ dv, int N, int d, int bq, int bk, int tm,
    int tn, int H, float inv_sqrt_d) {
    extern __shared__ float sm[];
    const int ld = MD + 1;
    float* sq = sm;                       // [rb][ld]   Q_i rows of this sub-block
    float* sdo = sq + bw::MAXB * ld;      // [rb][ld]   d_os = a dO
    float* sk = sdo + bw::MAXB * ld;      // [bk][ld]   K~_j
    float* sv = sk + bw::MAXB * ld;       // [bk][ld]   V_j
    float* sps = sv + bw::MAXB * ld;      // [rb][bk+1] P, then dS
    float* spp = sps + bw::MAXB * (bw::MAXB + 1);  // [rb][bk+1] P (kept for dV)
    float* sdq = spp + bw::MAXB * (bw::MAXB + 1);  // [rb][ld]   dq accumulator
    __shared__ int sfull;
    const int nsub = bq > bw::MAXB ? bq / bw::MAXB : 1;
    const int i = blockIdx.x / nsub, sub = blockIdx.x % nsub;
    const int rb = bq > bw::MAXB ? bw::MAXB : bq;  // rows in this CTA
    const int64_t bh = blockIdx.y;
    const int h_ = (int)(bh % H);
    const uint8_t* mrow = mask + (bh * tm + i) * (int64_t)tn;
    if (threadIdx.x == 0) sfull = 1;
    __syncthreads();
    for (int j = threadIdx.x; j < tn; j += blockDim.x)
        if (!mrow[j]) sfull = 0;
    __syncthreads();
    float a = 1.0f / (1.0f + expf(-rho[(int64_t)h_ * tm + i]));
    a = fminf(fmaxf(a, 1.17549435e-38f), 1.0f - 5.9604645e-08f);
    if (sfull) a = 1.0f;
    const int64_t r0 = bh * N + (int64_t)i * bq + (int64_t)sub * rb;
    for (int e = threadIdx.x; e < rb * d; e += blockDim.x) {
        const int r = e / d, c = e % d;
        sq[r * ld + c] = q[(r0 + r) * d + c];
        sdo[r * ld + c] = a * d_out[(r0 + r) * d + c];
        sdq[r * ld + c] = 0.0f;
    }
    const int pl = bw::MAXB + 1;
    for (int j = 0; j < tn; ++j) {
        if (!mrow[j]) continue;
        const int64_t c0 = bh * N + (int64_t)j * bk;
        __syncthreads();
        for (int e = threadIdx.x; e < bk * d; e += blockDim.x) {
            const int t = e / d, c = e % d;
            sk[t * ld + c] = k[(c0 + t) * d + c] - (mu ? mu[bh * d + c] : 0.0f);
            sv[t * ld + c] = v[(c0 + t) * d + c];
        }
        __syncthreads();
        // P = exp(S - L) (the hard weight is 1), dS = P (dP - rowsum(d_os o O_s)) / sqrt(d)
        for (int e = threadIdx.x; e < rb * bk; e += blockDim.x) {
            const int r = e / bk, t = e % bk;
            float s = 0.0f, dp = 0.0f;
            for (int f = 0; f < d; ++f) {
                s += sq[r * ld + f] * sk[t * ld + f];
                dp += sdo[r * ld + f] * sv[t * ld + f];
            }
            const float p = expf(s * inv_sqrt_d - big_l[r0 + r]);
            spp[r * pl + t] = p;
            sps[r * pl + t] = p * (dp - dsr[r0 + r]) * inv_sqrt_d;
        }
        __syncthreads();
        // dq_i += dS K~_j (owned); dK~_j += dS^T Q_i, dV_j += P^T d_os (atomic over query blocks)
        for (int e = threadIdx.x; e < rb * d; e += blockDim.x) {
            const int r = e / d, f = e % d;
            float acc = 0.0f;
            for (int t = 0; t < bk; ++t) acc += sps[r * pl + t] * sk[t * ld + f];
            sdq[r * ld + f] += acc;
        }
        for (int e = threadIdx.x; e < bk * d; e += blockDim.x) {
            const int t = e / d, f = e % d;
            float ak = 0.0f, avv = 0.0f;
            for (int r = 0; r < rb; ++r) {
                ak += sps[r * pl + t] * sq[r * ld + f];
                avv += spp[r * pl + t] * sdo[r * ld + f];
            }
            atomicAdd(&dkt[(c0 + t) * d + f], ak);
            atomicAdd(&dv[(c0 + t) * d + f], avv);
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rb * d; e += blockDim.x) {
        const int r = e / d, c = e % d;
        dq[(r0 + r) * d + c] += sdq[r * ld + c];  // after the linear part (bwd_qblock_kernel)
    }
}
template <int MD>
constexpr size_t bwd_sparse_smem() {
    return sizeof(float) * (5 * bw::MAXB * (MD + 1) + 2 * bw::MAXB * (bw::MAXB + 1));
}

// ---------------------------------------------------------------- per key block: linear branch
template <int MD>
__global__ void __launch_bounds__(256) bwd_keylin_kernel(const float* __restrict__ v, const float* __restrict__ phik,
                                                         const uint8_t* __restrict__ mask, const float* __restrict__ dh,
                                                         const float* __restrict__ dz, float* __restrict__ dkt,
                                                         float* __restrict__ dv, int N, int d, int bk, int tm, int tn) {
    constexpr int NU = MD / 32;
    extern __shared__ float klsm[];
    float(*sdh)[MD + 1] = reinterpret_cast<float(*)[MD + 1]>(klsm);  // [MD][MD + 1]
    float* sdz = klsm + MD * (MD + 1);                               // [MD]
    __shared__ uint8_t suse[1024];  // query blocks whose complement holds j (tm <= 1024)
    const int j = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // i contributes when j is not kept in row i and row i is not full (attention.hpp:722-727)
    for (int i = threadIdx.x; i < tm; i += blockDim.x) {
        const uint8_t* mrow = mask + (bh * tm + i) * (int64_t)tn;
        bool full = true;
        for (int jj = 0; jj < tn && full; ++jj) full = mrow[jj] != 0;
        suse[i] = (!full && !mrow[j]) ? 1 : 0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        float acc = 0.0f;
        for (int i = 0; i < tm; ++i)
            if (suse[i]) acc += dh[(bh * tm + i) * (int64_t)d * d + e];
        sdh[e / d][e % d] = acc;
    }
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
        float acc = 0.0f;
        for (int i = 0; i < tm; ++i)
            if (suse[i]) acc += dz[(bh * tm + i) * d + f];
        sdz[f] = acc;
    }
    __syncthreads();
    for (int t = warp; t < bk; t += 8) {  // one warp per key row, lane owns f / c = lane + 32 u
        const int64_t g = bh * N + (int64_t)j * bk + t;
        float vr[NU], pk[NU];
        for (int u = 0; u < NU; ++u) {
            const int c = lane + 32 * u;
            vr[u] = c < d ? v[g * d + c] : 0.0f;
            pk[u] = c < d ? phik[g * d + c] : 0.0f;
        }
        float dpk[NU], dot = 0.0f, dvv[NU];
        for (int u = 0; u < NU; ++u) {
            const int f = lane + 32 * u;
            float acc = f < d ? sdz[f] : 0.0f, accv = 0.0f;
            for (int c = 0; c < d; ++c) {
                const float vc = __shfl_sync(0xffffffffu, vr[c >> 5], c & 31);
                const float pc = __shfl_sync(0xffffffffu, pk[c >> 5], c & 31);
                if (f < d) {
                    acc += vc * sdh[f][c];   // dphi(K~)_t[f] = dz[f] + sum_c V[t][c] dh[f][c]
                    accv += pc * sdh[c][f];  // dV_t[f]      += sum_c phi(K~)[t][c] dh[c][f]
                }
            }
            dpk[u] = acc;
            dvv[u] = accv;
            dot += dpk[u] * pk[u];
        }
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        for (int u = 0; u < NU; ++u) {
            const int f = lane + 32 * u;
            if (f < d) {
                dkt[g * d + f] += pk[u] * (dpk[u] - dot);  // row_softmax_backward (matrix.hpp:160-169)
                dv[g * d + f] += dvv[u];
            }
        }
    }
}

template <int MD>
constexpr size_t bwd_keylin_smem() { return sizeof(float) * (MD * (MD + 1) + MD); }

// ---------------------------------------------------------------- dK = dK~ - colmean(dK~)
__global__ void bwd_smooth_kernel(float* __restrict__ dk, int N, int d) {
    const int64_t bh = blockIdx.x;
    __shared__ float smean[128];
    __shared__ float spart[bw::THREADS];
    const int parts = blockDim.x / d;  // d divides 256 for every supported d? use the general form
    const int c = threadIdx.x % d, p = threadIdx.x / d;
    float acc = 0.0f;
    if (p < parts)
        for (int r = p; r < N; r += parts) acc += dk[(bh * N + r) * d + c];
    spart[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < d) {
        float t = 0.0f;
        for (int q = 0; q < parts; ++q) t += spart[q * d + threadIdx.x];
        smean[threadIdx.x] = t * (1.0f / (float)N);
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)N * d; e += blockDim.x) dk[bh * N * d + e] -= smean[e % d];
}

cudaError_t launch_keyblock_linear(const float* k, const float* v, const float* mu, float* phik, float* h, float* z,
                                   int64_t BH, int N, int d, int bk, cudaStream_t st, int* launches) {
    if (d > 64 || bk > bw::MAXB) return cudaErrorInvalidValue;  // the stage-1 soft path (d <= 64)
    bwd_keyblock_kernel<64><<<dim3(N / bk, (unsigned)BH), 256, bwd_keyblock_smem<64>(), st>>>(k, v, mu, phik, h, z, N,
                                                                                            d, bk);
    ++*launches;
    return cudaGetLastError();
}

template <int MD>
static cudaError_t launch_backward_t(const BackwardLaunch& a, cudaStream_t st, int* launches) {
    const int tm = a.tm, tn = a.tn;
    const dim3 gk(tn, (unsigned)a.BH), gq(tm, (unsigned)a.BH);
    const float* mu = a.smooth ? a.mu : nullptr;
    if (a.smooth) {
        cudaError_t e = launch_colmean(a.k, nullptr, false, a.mu, (int)a.BH, a.N, a.d, st, launches);
        if (e != cudaSuccess) return e;
    }
    cudaMemsetAsync(a.dk, 0, sizeof(float) * a.BH * a.N * a.d, st);
    cudaMemsetAsync(a.dv, 0, sizeof(float) * a.BH * a.N * a.d, st);
    ensure_smem_attr((const void*)bwd_keyblock_kernel<MD>, (int)bwd_keyblock_smem<MD>());
    bwd_keyblock_kernel<MD><<<gk, 256, bwd_keyblock_smem<MD>(), st>>>(a.k, a.v, mu, a.phik, a.h, a.z, a.N, a.d, a.bk);
    bwd_total_kernel<<<dim3((a.d * a.d + 255) / 256, (unsigned)a.BH), 256, 0, st>>>(a.h, a.z, a.htot, a.ztot, tn, a.d);
    const size_t qsm = bwd_qblock_smem<MD>(a.bq);
    ensure_smem_attr((const void*)bwd_qblock_kernel<MD>, (int)qsm);
    bwd_qblock_kernel<MD><<<gq, 256, qsm, st>>>(a.q, a.d_out, a.o_s, a.o_l, a.mask, a.rho, a.h, a.z, a.htot, a.ztot,
                                                a.dq, a.dsr, a.dh, a.dz, a.drho, a.N, a.d, a.bq, tm, tn, (int)a.H);
    const int nsub = a.bq > bw::MAXB ? a.bq / bw::MAXB : 1;
    ensure_smem_attr((const void*)bwd_sparse_kernel<MD>, (int)bwd_sparse_smem<MD>());
    bwd_sparse_kernel<MD><<<dim3(tm * nsub, (unsigned)a.BH), 256, bwd_sparse_smem<MD>(), st>>>(
        a.q, a.k, a.v, mu, a.d_out, a.big_l, a.dsr, a.mask, a.rho, a.dq, a.dk, a.dv, a.N, a.d, a.bq, a.bk, tm, tn,
        (int)a.H, a.inv_sqrt_d);
    ensure_smem_attr((const void*)bwd_keylin_kernel<MD>, (int)bwd_keylin_smem<MD>());
    bwd_keylin_kernel<MD><<<gk, 256, bwd_keylin_smem<MD>(), st>>>(a.v, a.phik, a.mask, a.dh, a.dz, a.dk, a.dv, a.N,
                                                                  a.d, a.bk, tm, tn);
    if (a.smooth) bwd_smooth_kernel<<<(unsigned)a.BH, 256, 0, st>>>(a.dk, a.N, a.d);
    *launches += 5 + (a.smooth ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_backward(const BackwardLaunch& a, cudaStream_t st, int* launches) {
    if (a.d > 128 || a.bk > bw::MAXB || (a.bq > bw::MAXB && a.bq % bw::MAXB != 0) || a.tm > 1024 ||
        bwd_qblock_smem<128>(a.bq) > 227 * 1024)
        return cudaErrorInvalidValue;
    return a.d <= 64 ? launch_backward_t<64>(a, st, launches) : launch_backward_t<128>(a, st, launches);
}

}  // namespace sla2dev
