// sla2_b200/reference_dropin.hpp -- the B200 drop-in ON the reference's own types.
//
// Selected by sla2_b200/sla2.hpp when the reference headers (sla2/attention.hpp, ...) are on the
// include path. It includes them and adds EXPLICIT SPECIALIZATIONS of the reference's own
// function templates for T = float and T = double:
//
//   sla2::smooth_k<T>               quant.hpp:88-96
//   sla2::block_scores<T>           router.hpp:87-102
//   sla2::hard_topk<T>              router.hpp:106-125
//   sla2::sla2_forward_blockwise<T> attention.hpp:423-560 (BlockMask and SoftMask routing)
//
// so that every caller of those names in the translation unit -- Tape::sla2_attention
// (tape.hpp:263-286), model_forward (model.hpp:265-268), stage-1/2 training -- runs them on the
// B200 through the C ABI, with the reference's Matrix / Vector / RouterParams / BlockMask /
// MixRatio / AttentionInputs / SLA2ForwardSaved and its shape_error / numeric_error /
// contract_error. Nothing of the reference is redefined.
//
// ORDER: include this header (through sla2_b200/sla2.hpp) BEFORE sla2/tape.hpp,
// sla2/model.hpp, sla2/training.hpp: a specialization must be declared before the first use
// that would instantiate the template ([temp.expl.spec]/7). A translation unit that includes
// the drop-in must not be linked with one that instantiates the reference's own definitions of
// these four templates for the same T (the one-definition rule).
//
// Precision. The device computes in fp32 (b200::Precision::fp32, the default: CUDA-core
// kernels, the reference's float tolerance 1e-4) or bf16 (tcgen05 kernels, d = 128, bq = 128,
// bk = 64, tolerance 1e-2). T = float: the router is bit-exact with the reference. T = double
// (the Tape is double-only, tape.hpp:12-13): the matrices are rounded to float on the way in
// and widened on the way out, so the router is the reference's FLOAT router -- a mask can
// differ from the double reference's where two block scores agree to float precision.
//
// The saved state is complete (attention.hpp:345-358): o_s, o_l, big_l, h_blocks, z_blocks,
// q_phi, k_phi, routing, smoothed, bq, bk -- the reference's own sla2_backward consumes it
// unchanged (the backward itself stays the reference's: SURVEY.md 8(f) item 1;
// sla2::b200::backward_hard runs the device backward on request). On SoftMask routing
// h_blocks / z_blocks are not materialized (the stage-1 kernels do not form them): sized
// empty; o_s, o_l, big_l, q_phi, k_phi are filled.
//
// Not on the device (throws contract_error, as the C ABI reports): QuantConfig outside the
// bf16 kernel geometry (d = 128, bq = 128, bk = 64), SoftMask routing with d, bq or bk > 64.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "sla2/attention.hpp"
#include "sla2/quant.hpp"
#include "sla2/router.hpp"
#include "../sla2_capi.h"

#define SLA2_B200_REFERENCE_TYPES 1

namespace sla2 {
namespace b200 {

enum class Precision { fp32, bf16 };
inline Precision& precision() {
    static Precision p = Precision::fp32;
    return p;
}

// C ABI status -> the reference's exception classes (common.hpp:13-29)
inline void check(sla2_status s) {
    if (s == SLA2_OK) return;
    const std::string msg = sla2_last_error();
    if (s == SLA2_SHAPE_ERROR) throw shape_error(msg);
    if (s == SLA2_NUMERIC_ERROR) throw numeric_error(msg);
    if (s == SLA2_CONTRACT_ERROR) throw contract_error(msg);
    throw std::runtime_error("sla2_b200 CUDA error: " + msg);
}
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("sla2_b200: ") + what + ": " + cudaGetErrorString(e));
}

struct DeviceBuffer {  // owning device allocation
    void* p = nullptr;
    size_t n = 0;
    explicit DeviceBuffer(size_t bytes) : n(bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DeviceBuffer() {
        if (p) cudaFree(p);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    template <class U>
    U* as() const { return static_cast<U*>(p); }
};

// host T values -> device fp32 (T = double rounds to nearest) or bf16
template <class T>
inline void upload(DeviceBuffer& dst, const std::vector<T>& src, bool bf16 = false) {
    if (bf16) {
        std::vector<uint16_t> h(src.size());
        for (size_t i = 0; i < src.size(); ++i) {
            const float f = static_cast<float>(src[i]);
            uint32_t u;
            std::memcpy(&u, &f, 4);
            u += 0x7FFFu + ((u >> 16) & 1u);  // round to nearest even (finite inputs)
            h[i] = static_cast<uint16_t>(u >> 16);
        }
        cuda_check(cudaMemcpy(dst.p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "H2D");
        return;
    }
    if constexpr (std::is_same<T, float>::value) {
        cuda_check(cudaMemcpy(dst.p, src.data(), src.size() * 4, cudaMemcpyHostToDevice), "H2D");
    } else {
        std::vector<float> h(src.begin(), src.end());
        cuda_check(cudaMemcpy(dst.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "H2D");
    }
}
template <class T>
inline void download(std::vector<T>& dst, const void* src, size_t count, bool bf16 = false) {
    dst.resize(count);
    if (bf16) {
        std::vector<uint16_t> h(count);
        cuda_check(cudaMemcpy(h.data(), src, count * 2, cudaMemcpyDeviceToHost), "D2H");
        for (size_t i = 0; i < count; ++i) {
            const uint32_t u = static_cast<uint32_t>(h[i]) << 16;
            float f;
            std::memcpy(&f, &u, 4);
            dst[i] = static_cast<T>(f);
        }
        return;
    }
    std::vector<float> h(count);
    cuda_check(cudaMemcpy(h.data(), src, count * 4, cudaMemcpyDeviceToHost), "D2H");
    for (size_t i = 0; i < count; ++i) dst[i] = static_cast<T>(h[i]);
}
template <class T>
inline Matrix<T> download_matrix(const void* src, size_t r, size_t c, bool bf16 = false) {
    std::vector<T> v;
    download(v, src, r * c, bf16);
    return Matrix<T>(r, c, std::move(v));
}

inline sla2_fwd_params params(size_t n, size_t d, size_t bq, size_t bk, double k_percent, bool bf16, bool quant,
                              bool smooth) {
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)n, (int64_t)d);
    p.bq = (int64_t)bq;
    p.bk = (int64_t)bk;
    p.k_percent = k_percent;
    p.dtype = (bf16 || quant) ? SLA2_BF16 : SLA2_F32;
    p.quant = quant ? SLA2_QUANT_INT8 : SLA2_QUANT_NONE;
    p.smooth = smooth ? 1 : 0;
    return p;
}

template <class T>
inline std::pair<Matrix<T>, Vector<T>> smooth_k_impl(const Matrix<T>& k) {
    sla2_fwd_params p = params(k.rows(), k.cols(), 1, 1, 100.0, false, false, true);
    DeviceBuffer dk(k.size() * 4), dmu(k.cols() * 4);
    upload(dk, k.data());
    check(sla2_smooth_k(&p, dk.p, dmu.as<float>(), nullptr, nullptr));
    std::vector<T> mu;
    download(mu, dmu.p, k.cols());
    Matrix<T> out(k.rows(), k.cols());
    for (size_t i = 0; i < k.rows(); ++i)
        for (size_t j = 0; j < k.cols(); ++j) out(i, j) = k(i, j) - mu[j];
    return {std::move(out), Vector<T>(std::move(mu))};
}

template <class T>
inline Matrix<T> block_scores_impl(const Matrix<T>& q, const Matrix<T>& k, const RouterParams<T>& rp, size_t bq,
                                   size_t bk) {
    rp.validate();
    const size_t n = q.rows(), d = q.cols();
    if (k.cols() != d || rp.proj_q.rows() != d) throw shape_error("block_scores: feature dimension mismatch");
    if (bq == 0 || bk == 0 || n % bq || n % bk || k.rows() != n)
        throw shape_error("mean_pool: rows not divisible by block");
    sla2_fwd_params p = params(n, d, bq, bk, 100.0, false, false, false);
    p.tau = static_cast<float>(rp.tau);
    const size_t tm = n / bq, tn = n / bk;
    DeviceBuffer dq(n * d * 4), dk(n * d * 4), dpq(d * d * 4), dpk(d * d * 4), dpc(tm * tn * 4), dmask(tm * tn),
        didx(tm * tn * 4);
    upload(dq, q.data());
    upload(dk, k.data());
    upload(dpq, rp.proj_q.data());
    upload(dpk, rp.proj_k.data());
    const size_t ws = sla2_workspace_size(&p);
    if (!ws) check(sla2_check_params(&p));
    DeviceBuffer dws(ws);
    check(sla2_router(&p, dq.p, dk.p, dpq.as<float>(), dpk.as<float>(), dpc.as<float>(), dmask.as<uint8_t>(),
                      didx.as<int32_t>(), dws.p, ws, nullptr));
    return download_matrix<T>(dpc.p, tm, tn);
}

template <class T>
inline BlockMask hard_topk_impl(const Matrix<T>& pc, double k_percent) {
    if (!(k_percent > 0.0 && k_percent <= 100.0)) throw shape_error("hard_topk: k_percent must be in (0, 100]");
    const size_t tm = pc.rows(), tn = pc.cols();
    BlockMask mask = BlockMask::zeros(tm, tn);
    mask.keep_per_row = topk_budget(k_percent, tn);
    if (tm == 0 || tn == 0) return mask;
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)(tm * tn), 1);
    p.bq = (int64_t)tn;  // score-matrix geometry: rows N / bq = tm, columns N / bk = tn
    p.bk = (int64_t)tm;
    p.k_percent = k_percent;
    DeviceBuffer dpc(pc.size() * 4), dmask(tm * tn), didx(tm * mask.keep_per_row * 4 + 4);
    upload(dpc, pc.data());
    check(sla2_hard_topk(&p, dpc.as<float>(), dmask.as<uint8_t>(), didx.as<int32_t>(), nullptr));
    cuda_check(cudaMemcpy(mask.bits.data(), dmask.p, tm * tn, cudaMemcpyDeviceToHost), "D2H");
    return mask;
}

template <class T>
inline std::pair<Matrix<T>, SLA2ForwardSaved<T>> forward_impl(const AttentionInputs<T>& inputs,
                                                              const Routing<T>& routing, const MixRatio<T>& alpha,
                                                              const QuantConfig* quant, bool smooth) {
    inputs.validate();
    const size_t n = inputs.seq_len(), d = inputs.head_dim(), tm = inputs.tm(), tn = inputs.tn();
    if (alpha.rho.size() != tm) throw shape_error("sla2_forward_blockwise: rho length != tm");
    SLA2ForwardSaved<T> saved;
    saved.routing = routing;
    saved.smoothed = smooth;
    saved.bq = inputs.bq;
    saved.bk = inputs.bk;
    const size_t nd = n * d;
    DeviceBuffer dos(nd * 4), dol(nd * 4), dl(n * 4), dqphi(nd * 4), dkphi(nd * 4), drho(tm * 4);
    upload(drho, alpha.rho.data());
    bool bf16 = false;
    DeviceBuffer* dout_p = nullptr;
    if (std::holds_alternative<SoftMask<T>>(routing)) {
        // stage-1 SoftMask (attention.hpp:484-558): the fp32 stage-1 kernels
        const SoftMask<T>& soft = std::get<SoftMask<T>>(routing);
        if (soft.tm != tm || soft.tn != tn) throw shape_error("sla2_forward_blockwise: soft mask geometry mismatch");
        if (quant != nullptr) throw contract_error("sla2_forward_blockwise: SoftMask routing is full precision here");
        sla2_fwd_params p = params(n, d, inputs.bq, inputs.bk, 100.0, false, false, smooth);
        const size_t ws = sla2_forward_soft_workspace_size(&p);
        if (ws == 0)
            check(sla2_forward_soft(&p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                    nullptr));
        DeviceBuffer dq(nd * 4), dk(nd * 4), dv(nd * 4), dw(tm * tn * 4), dws(ws);
        DeviceBuffer dout(nd * 4);
        upload(dq, inputs.q.data());
        upload(dk, inputs.k.data());
        upload(dv, inputs.v.data());
        upload(dw, soft.values.data());
        sla2_fwd_saved sv{dos.as<float>(), dol.as<float>(), dl.as<float>(), nullptr, nullptr, nullptr, nullptr,
                          nullptr};
        check(sla2_forward_soft(&p, dq.p, dk.p, dv.p, drho.as<float>(), dw.as<float>(), dout.p, &sv, dws.p, ws,
                                nullptr));
        cuda_check(cudaDeviceSynchronize(), "sla2_forward_blockwise");
        Matrix<T> out = download_matrix<T>(dout.p, n, d);
        saved.o_s = download_matrix<T>(dos.p, n, d);
        saved.o_l = download_matrix<T>(dol.p, n, d);
        std::vector<T> bl;
        download(bl, dl.p, n);
        saved.big_l = Vector<T>(std::move(bl));
        // q_phi / k_phi: the hard path's exact feature maps of the same inputs
        BlockMask ones = BlockMask::ones(tm, tn);
        auto hard = forward_impl<T>(inputs, Routing<T>{ones}, alpha, nullptr, smooth);
        saved.q_phi = std::move(hard.second.q_phi);
        saved.k_phi = std::move(hard.second.k_phi);
        return {std::move(out), std::move(saved)};
    }
    const BlockMask& mask = std::get<BlockMask>(routing);
    if (mask.tm != tm || mask.tn != tn) throw shape_error("sla2_forward_blockwise: mask geometry mismatch");
    const bool q8 = quant != nullptr && (quant->qk_product || quant->pv_product);
    bf16 = precision() == Precision::bf16 || q8;
    sla2_fwd_params p = params(n, d, inputs.bq, inputs.bk, 100.0, bf16, q8, smooth);
    check(sla2_check_params(&p));
    const size_t esz = bf16 ? 2 : 4;
    DeviceBuffer dq(nd * esz), dk(nd * esz), dv(nd * esz), dout(nd * esz), dmask(tm * tn), dhb(tm * d * d * 4),
        dzb(tm * d * 4);
    dout_p = &dout;
    upload(dq, inputs.q.data(), bf16);
    upload(dk, inputs.k.data(), bf16);
    upload(dv, inputs.v.data(), bf16);
    cuda_check(cudaMemcpy(dmask.p, mask.bits.data(), tm * tn, cudaMemcpyHostToDevice), "H2D");
    const size_t ws = sla2_workspace_size(&p);
    DeviceBuffer dws(ws);
    sla2_fwd_saved sv{dos.as<float>(), dol.as<float>(), dl.as<float>(), dhb.as<float>(), dzb.as<float>(),
                      dqphi.as<float>(), dkphi.as<float>(), nullptr};
    // an empty mask row throws shape_error like attention.hpp:442-447
    check(sla2_sparse_fwd(&p, dq.p, dk.p, dv.p, drho.as<float>(), dmask.as<uint8_t>(), dout.p, &sv, dws.p, ws,
                          nullptr));
    cuda_check(cudaDeviceSynchronize(), "sla2_forward_blockwise");
    Matrix<T> out = download_matrix<T>(dout_p->p, n, d, bf16);
    saved.o_s = download_matrix<T>(dos.p, n, d);
    saved.o_l = download_matrix<T>(dol.p, n, d);
    std::vector<T> bl;
    download(bl, dl.p, n);
    saved.big_l = Vector<T>(std::move(bl));
    saved.q_phi = download_matrix<T>(dqphi.p, n, d);
    saved.k_phi = download_matrix<T>(dkphi.p, n, d);
    std::vector<T> hb, zb;
    download(hb, dhb.p, tm * d * d);
    download(zb, dzb.p, tm * d);
    saved.h_blocks.reserve(tm);
    saved.z_blocks.reserve(tm);
    for (size_t i = 0; i < tm; ++i) {
        saved.h_blocks.emplace_back(d, d, std::vector<T>(hb.begin() + i * d * d, hb.begin() + (i + 1) * d * d));
        saved.z_blocks.emplace_back(std::vector<T>(zb.begin() + i * d, zb.begin() + (i + 1) * d));
    }
    return {std::move(out), std::move(saved)};
}

// The device backward (sla2_backward C ABI: hard routing, fp32, d <= 128, bk <= 64, bq <= 64 or 128) on request; the
// reference's own sla2_backward stays in place for everything else.
template <class T>
inline SLA2Gradients<T> backward_hard(const SLA2ForwardSaved<T>& saved, const AttentionInputs<T>& inputs,
                                      const MixRatio<T>& alpha, const Matrix<T>& d_out) {
    inputs.validate();
    const size_t n = inputs.seq_len(), d = inputs.head_dim(), tm = inputs.tm(), tn = inputs.tn();
    if (saved.o_s.rows() != n || saved.o_s.cols() != d || saved.big_l.size() != n)
        throw contract_error("sla2_backward: saved state missing or inconsistent");  // attention.hpp:620-622
    if (!d_out.same_shape(saved.o_s)) throw shape_error("sla2_backward: d_out shape mismatch");
    if (!saved.hard()) throw contract_error("sla2_backward: SoftMask routing is not on the device backward");
    const BlockMask& mask = std::get<BlockMask>(saved.routing);
    sla2_fwd_params p = params(n, d, inputs.bq, inputs.bk, 100.0, false, false, saved.smoothed);
    const size_t ws = sla2_backward_workspace_size(&p);
    if (ws == 0)
        check(sla2_backward(&p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr));
    const size_t nd = n * d * 4;
    DeviceBuffer dq(nd), dk(nd), dv(nd), ddo(nd), dos(nd), dol(nd), dl(n * 4), drho(tm * 4), dmask(tm * tn), gq(nd),
        gk(nd), gv(nd), grho(tm * 4), dws(ws);
    upload(dq, inputs.q.data());
    upload(dk, inputs.k.data());
    upload(dv, inputs.v.data());
    upload(ddo, d_out.data());
    upload(dos, saved.o_s.data());
    upload(dol, saved.o_l.data());
    upload(dl, saved.big_l.data());
    upload(drho, alpha.rho.data());
    cuda_check(cudaMemcpy(dmask.p, mask.bits.data(), tm * tn, cudaMemcpyHostToDevice), "H2D");
    check(sla2_backward(&p, dq.p, dk.p, dv.p, drho.as<float>(), dmask.as<uint8_t>(), dos.as<float>(), dol.as<float>(),
                        dl.as<float>(), ddo.p, gq.p, gk.p, gv.p, grho.as<float>(), dws.p, ws, nullptr));
    cuda_check(cudaDeviceSynchronize(), "sla2_backward");
    SLA2Gradients<T> g;
    g.dq = download_matrix<T>(gq.p, n, d);
    g.dk = download_matrix<T>(gk.p, n, d);
    g.dv = download_matrix<T>(gv.p, n, d);
    std::vector<T> dr;
    download(dr, grho.p, tm);
    g.drho = Vector<T>(std::move(dr));
    return g;
}

// Tape::sla2_attention's forward composition (tape.hpp:263-272) on plain matrices -- the same
// helper the standalone header offers: smooth_k -> block_scores(q, K~) -> hard_topk ->
// sla2_forward_blockwise, every step on the device.
template <class T>
inline Matrix<T> sla2_attention(const Matrix<T>& q, const Matrix<T>& k, const Matrix<T>& v, const MixRatio<T>& mix,
                                const RouterParams<T>& router, size_t bq, size_t bk, double k_percent,
                                const QuantConfig* quant = nullptr, bool smooth = true, BlockMask* mask_out = nullptr) {
    AttentionInputs<T> in{q, k, v, bq, bk};
    const Matrix<T> ktilde = smooth ? smooth_k_impl<T>(k).first : k;
    BlockMask mask = hard_topk_impl<T>(block_scores_impl<T>(q, ktilde, router, bq, bk), k_percent);
    if (mask_out) *mask_out = mask;
    return forward_impl<T>(in, Routing<T>{std::move(mask)}, mix, quant, smooth).first;
}

}  // namespace b200

// ---------------------------------------------------------------- the specializations
#define SLA2_B200_SPECIALIZE(T)                                                                              \
    template <>                                                                                              \
    inline std::pair<Matrix<T>, Vector<T>> smooth_k<T>(const Matrix<T>& k) {                                 \
        return b200::smooth_k_impl<T>(k);                                                                    \
    }                                                                                                        \
    template <>                                                                                              \
    inline Matrix<T> block_scores<T>(const Matrix<T>& q, const Matrix<T>& k, const RouterParams<T>& params,  \
                                     std::size_t bq, std::size_t bk) {                                       \
        return b200::block_scores_impl<T>(q, k, params, bq, bk);                                             \
    }                                                                                                        \
    template <>                                                                                              \
    inline BlockMask hard_topk<T>(const Matrix<T>& pc, double k_percent) {                                   \
        return b200::hard_topk_impl<T>(pc, k_percent);                                                       \
    }                                                                                                        \
    template <>                                                                                              \
    inline std::pair<Matrix<T>, SLA2ForwardSaved<T>> sla2_forward_blockwise<T>(                              \
        const AttentionInputs<T>& inputs, const Routing<T>& routing, const MixRatio<T>& alpha,               \
        const QuantConfig* quant, bool smooth) {                                                             \
        return b200::forward_impl<T>(inputs, routing, alpha, quant, smooth);                                 \
    }
SLA2_B200_SPECIALIZE(float)
SLA2_B200_SPECIALIZE(double)
#undef SLA2_B200_SPECIALIZE

}  // namespace sla2
