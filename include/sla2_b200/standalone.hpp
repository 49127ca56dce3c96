// sla2_b200/standalone.hpp -- the drop-in without the reference headers (selected by
// sla2_b200/sla2.hpp when sla2/attention.hpp is not on the include path): mirrors of the
// reference's types and entry points on the C ABI.
//
// A caller of the reference library (/root/reference/proj/include/sla2/*.hpp) switches to the
// B200 implementation by including this header instead of sla2/router.hpp + sla2/quant.hpp +
// sla2/attention.hpp and linking libsla2_b200.so (+ libcudart). The names, signatures,
// argument meaning, value semantics and exception classes below are the reference's:
//
//   sla2::topk_budget             router.hpp:36-40
//   sla2::smooth_k                quant.hpp:88-96
//   sla2::block_scores            router.hpp:87-102
//   sla2::hard_topk               router.hpp:106-125
//   sla2::sla2_forward_blockwise  attention.hpp:423-560   (hard BlockMask routing)
//   sla2::sla2_attention          the forward composition of Tape::sla2_attention,
//                                 tape.hpp:263-272 (no autodiff tape on the B200 path)
//   sla2::shape_error / numeric_error / contract_error   common.hpp:13-29
//
// Element type: float (Matrix<float>), the reference's "production" precision
// (SPEC.md:77). Computation happens on the current CUDA device through the C ABI; inputs and
// outputs stay host matrices, as in the reference. Precision::fp32 (default) runs the fp32
// CUDA-core kernels (reference tolerance 1e-4); Precision::bf16 rounds Q/K/V to bf16 and runs
// the tcgen05 kernels (d = 128, bq = 128, bk = 64; tolerance 1e-2). The router (smooth_k,
// block_scores, hard_topk) is bit-exact with the reference in both.
// Not on this path (throws contract_error): SoftMask routing (stage-1 training), double.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <type_traits>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "../sla2_capi.h"

namespace sla2 {

// ------------------------------------------------------------------ errors (common.hpp:13-29)
class shape_error : public std::invalid_argument {
public:
    explicit shape_error(const std::string& what) : std::invalid_argument(what) {}
};
class numeric_error : public std::runtime_error {
public:
    explicit numeric_error(const std::string& what) : std::runtime_error(what) {}
};
class contract_error : public std::runtime_error {
public:
    explicit contract_error(const std::string& what) : std::runtime_error(what) {}
};

namespace b200 {
enum class Precision { fp32, bf16 };
inline Precision& precision() {
    static Precision p = Precision::fp32;
    return p;
}
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
// Owning device buffer.
struct DeviceBuffer {
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
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void upload(const void* src, size_t bytes) { cuda_check(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "H2D"); }
    void download(void* dst, size_t bytes) const {
        cuda_check(cudaMemcpy(dst, p, bytes, cudaMemcpyDeviceToHost), "D2H");
    }
};
}  // namespace b200

// ------------------------------------------------------------------ carriers (matrix.hpp:18-97)
template <class T>
class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, T fill = T(0)) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    Matrix(std::size_t rows, std::size_t cols, std::vector<T> data)
        : rows_(rows), cols_(cols), data_(std::move(data)) {
        if (rows_ * cols_ != data_.size()) throw shape_error("Matrix: rows*cols != data length");
        check_finite("Matrix construction");
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    T& operator()(std::size_t r, std::size_t c) { return data_[r * cols_ + c]; }
    const T& operator()(std::size_t r, std::size_t c) const { return data_[r * cols_ + c]; }
    std::vector<T>& data() { return data_; }
    const std::vector<T>& data() const { return data_; }
    bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
    void check_finite(const char* where) const {
        for (const T v : data_)
            if (!std::isfinite(v)) throw numeric_error(std::string(where) + ": non-finite entry");
    }
    static Matrix identity(std::size_t n) {
        Matrix m(n, n, T(0));
        for (std::size_t i = 0; i < n; ++i) m(i, i) = T(1);
        return m;
    }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<T> data_;
};

template <class T>
class Vector {
public:
    Vector() = default;
    explicit Vector(std::size_t len, T fill = T(0)) : data_(len, fill) {}
    explicit Vector(std::vector<T> data) : data_(std::move(data)) {}
    std::size_t size() const { return data_.size(); }
    T& operator[](std::size_t i) { return data_[i]; }
    const T& operator[](std::size_t i) const { return data_[i]; }
    std::vector<T>& data() { return data_; }
    const std::vector<T>& data() const { return data_; }

private:
    std::vector<T> data_;
};

// ------------------------------------------------------------------ router types (router.hpp)
template <class T>
struct RouterParams {
    Matrix<T> proj_q, proj_k;
    T tau = T(0.1);
    static RouterParams identity(std::size_t d, T tau = T(0.1)) {
        return RouterParams{Matrix<T>::identity(d), Matrix<T>::identity(d), tau};
    }
    void validate() const {
        if (proj_q.rows() != proj_q.cols() || proj_k.rows() != proj_k.cols() || proj_q.rows() != proj_k.rows())
            throw shape_error("RouterParams: projections must be square with equal side");
        if (!(tau > T(0))) throw numeric_error("RouterParams: tau must be positive");
    }
};

struct BlockMask {
    std::size_t tm = 0, tn = 0;
    std::vector<std::uint8_t> bits;
    std::size_t keep_per_row = 0;
    std::uint8_t at(std::size_t i, std::size_t j) const { return bits[i * tn + j]; }
    std::uint8_t& at(std::size_t i, std::size_t j) { return bits[i * tn + j]; }
    double sparsity() const {
        std::size_t ones = 0;
        for (const auto b : bits) ones += b;
        return 1.0 - static_cast<double>(ones) / static_cast<double>(tm * tn);
    }
    bool row_full(std::size_t i) const {
        for (std::size_t j = 0; j < tn; ++j)
            if (!at(i, j)) return false;
        return true;
    }
    static BlockMask ones(std::size_t tm, std::size_t tn) { return BlockMask{tm, tn, std::vector<std::uint8_t>(tm * tn, 1), tn}; }
    static BlockMask zeros(std::size_t tm, std::size_t tn) { return BlockMask{tm, tn, std::vector<std::uint8_t>(tm * tn, 0), 0}; }
};

// Stage-1 soft routing (router.hpp:74-82): soft_topk and the SoftMask forward run on the device
// (sla2_soft_topk / sla2_forward_soft, fp32); the soft backward is not on this path.
template <class T>
struct SoftMask {
    std::size_t tm = 0, tn = 0;
    Matrix<T> values;
    Vector<T> lambdas;
    T tau = T(0.1);
    std::size_t budget = 0;
};
template <class T>
using Routing = std::variant<BlockMask, SoftMask<T>>;

struct QuantConfig {  // quant.hpp:15-19
    int bits = 8;
    bool qk_product = true;
    bool pv_product = true;
};

template <class T>
T sigmoid(T x) {  // attention.hpp:17-22
    const T v = T(1) / (T(1) + std::exp(-x));
    const T lo = std::numeric_limits<T>::min(), hi = T(1) - std::numeric_limits<T>::epsilon() / 2;
    return v < lo ? lo : (v > hi ? hi : v);
}

template <class T>
struct MixRatio {  // attention.hpp:45-57
    Vector<T> rho;
    static MixRatio zeros(std::size_t tm) { return MixRatio{Vector<T>(tm, T(0))}; }
    static MixRatio constant(std::size_t tm, T v) { return MixRatio{Vector<T>(tm, v)}; }
    T alpha(std::size_t block) const { return sigmoid(rho[block]); }
};

template <class T>
struct AttentionInputs {  // attention.hpp:24-43
    Matrix<T> q, k, v;
    std::size_t bq = 1, bk = 1;
    std::size_t seq_len() const { return q.rows(); }
    std::size_t head_dim() const { return q.cols(); }
    std::size_t tm() const { return q.rows() / bq; }
    std::size_t tn() const { return q.rows() / bk; }
    void validate() const {
        if (!q.same_shape(k) || !q.same_shape(v)) throw shape_error("AttentionInputs: q, k, v must share N×d");
        if (bq == 0 || bk == 0 || q.rows() % bq != 0 || q.rows() % bk != 0)
            throw shape_error("AttentionInputs: N must be divisible by bq and bk");
    }
};

// What the B200 forward can return of SLA2ForwardSaved (attention.hpp:345-358): the branch
// outputs and the logsumexp. The per-block H_i/Z_i and phi maps are not materialized.
template <class T>
struct SLA2ForwardSaved {
    Matrix<T> o_s, o_l;
    Vector<T> big_l;
    Routing<T> routing;
    bool smoothed = true;
    std::size_t bq = 1, bk = 1;
    bool hard() const { return std::holds_alternative<BlockMask>(routing); }
};

namespace b200 {
inline sla2_fwd_params params(std::size_t n, std::size_t d, std::size_t bq, std::size_t bk, double k_percent,
                              bool quant, bool smooth) {
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)n, (int64_t)d);
    p.bq = (int64_t)bq;
    p.bk = (int64_t)bk;
    p.k_percent = k_percent;
    p.dtype = (precision() == Precision::bf16 || quant) ? SLA2_BF16 : SLA2_F32;
    p.quant = quant ? SLA2_QUANT_INT8 : SLA2_QUANT_NONE;
    p.smooth = smooth ? 1 : 0;
    return p;
}
// Upload a float matrix as the dtype p selects.
inline void upload_as(DeviceBuffer& dst, const Matrix<float>& m, const sla2_fwd_params& p) {
    if (p.dtype == SLA2_F32) {
        dst.upload(m.data().data(), m.size() * 4);
    } else {
        std::vector<__nv_bfloat16> h(m.size());
        for (std::size_t i = 0; i < m.size(); ++i) h[i] = __float2bfloat16_rn(m.data()[i]);
        dst.upload(h.data(), h.size() * 2);
    }
}
inline Matrix<float> download_as(const DeviceBuffer& src, std::size_t r, std::size_t c, const sla2_fwd_params& p) {
    Matrix<float> m(r, c);
    if (p.dtype == SLA2_F32) {
        src.download(m.data().data(), m.size() * 4);
    } else {
        std::vector<__nv_bfloat16> h(m.size());
        src.download(h.data(), h.size() * 2);
        for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = __bfloat162float(h[i]);
    }
    return m;
}
}  // namespace b200

// ------------------------------------------------------------------ operations
inline std::size_t topk_budget(double k_percent, std::size_t tn) {
    return static_cast<std::size_t>(sla2_topk_budget(k_percent, static_cast<int64_t>(tn)));
}

// quant.hpp:88-96. The column mean runs on the device in the reference's serial order.
inline std::pair<Matrix<float>, Vector<float>> smooth_k(const Matrix<float>& k) {
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)k.rows(), (int64_t)k.cols());
    p.bq = p.bk = 1;
    p.dtype = SLA2_F32;
    b200::DeviceBuffer dk(k.size() * 4), dmu(k.cols() * 4);
    dk.upload(k.data().data(), k.size() * 4);
    b200::check(sla2_smooth_k(&p, dk.p, dmu.as<float>(), nullptr, nullptr));
    Vector<float> mean(k.cols());
    dmu.download(mean.data().data(), k.cols() * 4);
    Matrix<float> out(k.rows(), k.cols());
    for (std::size_t i = 0; i < k.rows(); ++i)
        for (std::size_t j = 0; j < k.cols(); ++j) out(i, j) = k(i, j) - mean[j];
    return {std::move(out), std::move(mean)};
}

// router.hpp:87-102 (k is whatever the caller passes -- the reference's callers pass K~).
inline Matrix<float> block_scores(const Matrix<float>& q, const Matrix<float>& k, const RouterParams<float>& params,
                                  std::size_t bq, std::size_t bk) {
    params.validate();
    const std::size_t n = q.rows(), d = q.cols();
    if (k.cols() != d || params.proj_q.rows() != d) throw shape_error("block_scores: feature dimension mismatch");
    if (bq == 0 || bk == 0 || n % bq || n % bk || k.rows() != n)
        throw shape_error("mean_pool: rows not divisible by block");
    sla2_fwd_params p = b200::params(n, d, bq, bk, 100.0, false, false);
    p.dtype = SLA2_F32;  // the router is exact arithmetic on the float values given
    p.tau = params.tau;
    const std::size_t tm = n / bq, tn = n / bk;
    b200::DeviceBuffer dq(q.size() * 4), dk(k.size() * 4), dpq(d * d * 4), dpk(d * d * 4);
    b200::DeviceBuffer dpc(tm * tn * 4), dmask(tm * tn), didx(tm * tn * 4);
    dq.upload(q.data().data(), q.size() * 4);
    dk.upload(k.data().data(), k.size() * 4);
    dpq.upload(params.proj_q.data().data(), d * d * 4);
    dpk.upload(params.proj_k.data().data(), d * d * 4);
    size_t ws = sla2_workspace_size(&p);
    if (!ws) b200::check(sla2_check_params(&p));
    b200::DeviceBuffer dws(ws);
    b200::check(sla2_router(&p, dq.p, dk.p, dpq.as<float>(), dpk.as<float>(), dpc.as<float>(), dmask.as<uint8_t>(),
                            didx.as<int32_t>(), dws.p, ws, nullptr));
    Matrix<float> pc(tm, tn);
    dpc.download(pc.data().data(), tm * tn * 4);
    return pc;
}

// router.hpp:106-125
inline BlockMask hard_topk(const Matrix<float>& pc, double k_percent) {
    if (!(k_percent > 0.0 && k_percent <= 100.0)) throw shape_error("hard_topk: k_percent must be in (0, 100]");
    const std::size_t tm = pc.rows(), tn = pc.cols();
    BlockMask mask = BlockMask::zeros(tm, tn);
    mask.keep_per_row = topk_budget(k_percent, tn);
    if (tm == 0 || tn == 0) return mask;
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)(tm * tn), 1);
    p.bq = (int64_t)tn;  // rows = N / bq = tm
    p.bk = (int64_t)tm;  // cols = N / bk = tn
    p.k_percent = k_percent;
    b200::DeviceBuffer dpc(pc.size() * 4), dmask(tm * tn), didx(tm * mask.keep_per_row * 4 + 4);
    dpc.upload(pc.data().data(), pc.size() * 4);
    b200::check(sla2_hard_topk(&p, dpc.as<float>(), dmask.as<uint8_t>(), didx.as<int32_t>(), nullptr));
    dmask.download(mask.bits.data(), tm * tn);
    return mask;
}

// soft_topk (router.hpp:126-190) on the device: bisection in double per row, fp32 values.
inline SoftMask<float> soft_topk(const Matrix<float>& pc, double k_percent, float tau) {
    if (!(tau > 0.0f)) throw numeric_error("soft_topk: tau must be positive");
    const std::size_t tm = pc.rows(), tn = pc.cols();
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)(tm * tn), 1);  // only the tm x tn geometry is read
    p.bq = (int64_t)tn;
    p.bk = (int64_t)tm;
    p.k_percent = k_percent;
    p.dtype = SLA2_F32;
    p.tau = tau;
    SoftMask<float> out;
    out.tm = tm;
    out.tn = tn;
    out.tau = tau;
    out.budget = topk_budget(k_percent, tn);
    out.values = Matrix<float>(tm, tn);
    out.lambdas = Vector<float>(tm);
    b200::DeviceBuffer dpc(pc.size() * 4), dv(pc.size() * 4), dl(tm * 4);
    dpc.upload(pc.data().data(), pc.size() * 4);
    b200::check(sla2_soft_topk(&p, dpc.as<float>(), dv.as<float>(), dl.as<float>(), nullptr));
    dv.download(out.values.data().data(), pc.size() * 4);
    dl.download(out.lambdas.data().data(), tm * 4);
    return out;
}

// soft_topk_backward (router.hpp:197-212) on the device: upstream * v * (1 - v) / tau.
inline Matrix<float> soft_topk_backward(const Matrix<float>& pc, const SoftMask<float>& softmask,
                                        const Matrix<float>& upstream) {
    if (pc.rows() != softmask.tm || pc.cols() != softmask.tn || !pc.same_shape(upstream))
        throw shape_error("soft_topk_backward: shape mismatch");
    const std::size_t tm = pc.rows(), tn = pc.cols();
    sla2_fwd_params p;
    sla2_default_params(&p, 1, 1, (int64_t)(tm * tn), 1);
    p.bq = (int64_t)tn;
    p.bk = (int64_t)tm;
    p.dtype = SLA2_F32;
    p.tau = softmask.tau;
    b200::DeviceBuffer dv(pc.size() * 4), du(pc.size() * 4), dg(pc.size() * 4);
    dv.upload(softmask.values.data().data(), pc.size() * 4);
    du.upload(upstream.data().data(), pc.size() * 4);
    b200::check(sla2_soft_topk_backward(&p, dv.as<float>(), du.as<float>(), dg.as<float>(), nullptr));
    Matrix<float> grad(tm, tn);
    dg.download(grad.data().data(), pc.size() * 4);
    return grad;
}

// attention.hpp:423-560 (hard routing on the tcgen05 / fp32 kernels; SoftMask on the fp32
// stage-1 kernels).
inline std::pair<Matrix<float>, SLA2ForwardSaved<float>> sla2_forward_blockwise(const AttentionInputs<float>& inputs,
                                                                                const Routing<float>& routing,
                                                                                const MixRatio<float>& alpha,
                                                                                const QuantConfig* quant = nullptr,
                                                                                bool smooth = true) {
    inputs.validate();
    const std::size_t n = inputs.seq_len(), d = inputs.head_dim(), tm = inputs.tm(), tn = inputs.tn();
    if (alpha.rho.size() != tm) throw shape_error("sla2_forward_blockwise: rho length != tm");
    if (!std::holds_alternative<BlockMask>(routing)) {
        // SoftMask (attention.hpp:484-558): the fp32 stage-1 kernels, whatever precision() says
        const SoftMask<float>& soft = std::get<SoftMask<float>>(routing);
        if (soft.tm != tm || soft.tn != tn) throw shape_error("sla2_forward_blockwise: soft mask geometry mismatch");
        if (quant != nullptr) throw contract_error("sla2_forward_blockwise: SoftMask routing is full precision");
        sla2_fwd_params p = b200::params(n, d, inputs.bq, inputs.bk, 100.0, false, smooth);
        p.dtype = SLA2_F32;
        const size_t ws = sla2_forward_soft_workspace_size(&p);
        if (ws == 0)
            b200::check(sla2_forward_soft(&p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                          nullptr));
        b200::DeviceBuffer dq(n * d * 4), dk(n * d * 4), dv(n * d * 4), dout(n * d * 4), drho(tm * 4),
            dw(tm * tn * 4), dos(n * d * 4), dol(n * d * 4), dl(n * 4), dws(ws);
        dq.upload(inputs.q.data().data(), n * d * 4);
        dk.upload(inputs.k.data().data(), n * d * 4);
        dv.upload(inputs.v.data().data(), n * d * 4);
        drho.upload(alpha.rho.data().data(), tm * 4);
        dw.upload(soft.values.data().data(), tm * tn * 4);
        sla2_fwd_saved sv{dos.as<float>(), dol.as<float>(), dl.as<float>()};
        b200::check(sla2_forward_soft(&p, dq.p, dk.p, dv.p, drho.as<float>(), dw.as<float>(), dout.p, &sv, dws.p, ws,
                                      nullptr));
        b200::cuda_check(cudaDeviceSynchronize(), "sla2_forward_blockwise");
        SLA2ForwardSaved<float> saved;
        saved.routing = routing;
        saved.smoothed = smooth;
        saved.bq = inputs.bq;
        saved.bk = inputs.bk;
        saved.o_s = Matrix<float>(n, d);
        saved.o_l = Matrix<float>(n, d);
        saved.big_l = Vector<float>(n);
        Matrix<float> out(n, d);
        dout.download(out.data().data(), n * d * 4);
        dos.download(saved.o_s.data().data(), n * d * 4);
        dol.download(saved.o_l.data().data(), n * d * 4);
        dl.download(saved.big_l.data().data(), n * 4);
        return {std::move(out), std::move(saved)};
    }
    const BlockMask& mask = std::get<BlockMask>(routing);
    if (mask.tm != tm || mask.tn != tn) throw shape_error("sla2_forward_blockwise: mask geometry mismatch");
    for (std::size_t i = 0; i < tm; ++i) {
        bool any = false;
        for (std::size_t j = 0; j < tn; ++j) any |= mask.at(i, j) != 0;
        if (!any) throw shape_error("sla2_forward_blockwise: mask row keeps no blocks");
    }
    const bool q8 = quant != nullptr && (quant->qk_product || quant->pv_product);
    sla2_fwd_params p = b200::params(n, d, inputs.bq, inputs.bk, 100.0, q8, smooth);
    b200::check(sla2_check_params(&p));
    const std::size_t esz = p.dtype == SLA2_F32 ? 4 : 2;
    b200::DeviceBuffer dq(n * d * esz), dk(n * d * esz), dv(n * d * esz), dout(n * d * esz);
    b200::DeviceBuffer drho(tm * 4), dmask(tm * tn), dos(n * d * 4), dol(n * d * 4), dl(n * 4);
    b200::upload_as(dq, inputs.q, p);
    b200::upload_as(dk, inputs.k, p);
    b200::upload_as(dv, inputs.v, p);
    drho.upload(alpha.rho.data().data(), tm * 4);
    dmask.upload(mask.bits.data(), tm * tn);
    const size_t ws = sla2_workspace_size(&p);
    b200::DeviceBuffer dws(ws);
    sla2_fwd_saved sv{dos.as<float>(), dol.as<float>(), dl.as<float>()};
    b200::check(sla2_sparse_fwd(&p, dq.p, dk.p, dv.p, drho.as<float>(), dmask.as<uint8_t>(), dout.p, &sv, dws.p, ws,
                                nullptr));
    b200::cuda_check(cudaDeviceSynchronize(), "sla2_forward_blockwise");
    SLA2ForwardSaved<float> saved;
    saved.routing = routing;
    saved.smoothed = smooth;
    saved.bq = inputs.bq;
    saved.bk = inputs.bk;
    saved.o_s = Matrix<float>(n, d);
    saved.o_l = Matrix<float>(n, d);
    saved.big_l = Vector<float>(n);
    dos.download(saved.o_s.data().data(), n * d * 4);
    dol.download(saved.o_l.data().data(), n * d * 4);
    dl.download(saved.big_l.data().data(), n * 4);
    return {b200::download_as(dout, n, d, p), std::move(saved)};
}

// ------------------------------------------------------------------ backward (attention.hpp:562-809)
template <class T>
struct SLA2Gradients {
    Matrix<T> dq, dk, dv;
    Vector<T> drho;
    Matrix<T> dproj_q, dproj_k;  // stage-1 soft routing only: not on this path (left empty)
};

// sla2_backward on the hard-routing path (the stage-2 / QAT fine-tuning backward): full
// precision on the device from the forward's saved O_s, O_l, L and the mask. d <= 128, bk <= 64, bq <= 64 or 128.
inline SLA2Gradients<float> sla2_backward(const SLA2ForwardSaved<float>& saved, const AttentionInputs<float>& inputs,
                                          const MixRatio<float>& alpha, const Matrix<float>& d_out) {
    inputs.validate();
    const std::size_t n = inputs.seq_len(), d = inputs.head_dim(), tm = inputs.tm(), tn = inputs.tn();
    if (saved.o_s.rows() != n || saved.o_s.cols() != d || saved.big_l.size() != n)
        throw contract_error("sla2_backward: saved state missing or inconsistent");  // attention.hpp:620-622
    if (!d_out.same_shape(saved.o_s)) throw shape_error("sla2_backward: d_out shape mismatch");
    if (!saved.hard())
        throw contract_error("sla2_backward: SoftMask routing (stage-1 training) is not on the B200 path");
    if (alpha.rho.size() != tm) throw shape_error("sla2_backward: rho length != tm");
    const BlockMask& mask = std::get<BlockMask>(saved.routing);
    sla2_fwd_params p = b200::params(n, d, inputs.bq, inputs.bk, 100.0, false, saved.smoothed);
    p.dtype = SLA2_F32;  // the backward is full precision
    const size_t ws = sla2_backward_workspace_size(&p);
    if (ws == 0) b200::check(sla2_backward(&p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                           nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr));
    const size_t nd = n * d * 4;
    b200::DeviceBuffer dq(nd), dk(nd), dv(nd), ddo(nd), dos(nd), dol(nd), dl(n * 4), drho(tm * 4), dmask(tm * tn);
    b200::DeviceBuffer gq(nd), gk(nd), gv(nd), grho(tm * 4), dws(ws);
    dq.upload(inputs.q.data().data(), nd);
    dk.upload(inputs.k.data().data(), nd);
    dv.upload(inputs.v.data().data(), nd);
    ddo.upload(d_out.data().data(), nd);
    dos.upload(saved.o_s.data().data(), nd);
    dol.upload(saved.o_l.data().data(), nd);
    dl.upload(saved.big_l.data().data(), n * 4);
    drho.upload(alpha.rho.data().data(), tm * 4);
    dmask.upload(mask.bits.data(), tm * tn);
    b200::check(sla2_backward(&p, dq.p, dk.p, dv.p, drho.as<float>(), dmask.as<uint8_t>(), dos.as<float>(),
                              dol.as<float>(), dl.as<float>(), ddo.p, gq.p, gk.p, gv.p, grho.as<float>(), dws.p, ws,
                              nullptr));
    b200::cuda_check(cudaDeviceSynchronize(), "sla2_backward");
    SLA2Gradients<float> g;
    g.dq = Matrix<float>(n, d);
    g.dk = Matrix<float>(n, d);
    g.dv = Matrix<float>(n, d);
    g.drho = Vector<float>(tm);
    gq.download(g.dq.data().data(), nd);
    gk.download(g.dk.data().data(), nd);
    gv.download(g.dv.data().data(), nd);
    grho.download(g.drho.data().data(), tm * 4);
    return g;
}

// Tape::sla2_attention's forward composition (tape.hpp:263-272) on the device:
// smooth_k -> block_scores(q, K~) -> hard_topk -> sla2_forward_blockwise.
inline Matrix<float> sla2_attention(const Matrix<float>& q, const Matrix<float>& k, const Matrix<float>& v,
                                    const MixRatio<float>& mix, const RouterParams<float>& router, std::size_t bq,
                                    std::size_t bk, double k_percent, const QuantConfig* quant = nullptr,
                                    bool smooth = true, BlockMask* mask_out = nullptr) {
    router.validate();
    AttentionInputs<float> in{q, k, v, bq, bk};
    in.validate();
    const std::size_t n = q.rows(), d = q.cols(), tm = n / bq, tn = n / bk;
    if (mix.rho.size() != tm) throw shape_error("sla2_attention: rho length != tm");
    if (!(k_percent > 0.0 && k_percent <= 100.0)) throw shape_error("hard_topk: k_percent must be in (0, 100]");
    const bool q8 = quant != nullptr && (quant->qk_product || quant->pv_product);
    sla2_fwd_params p = b200::params(n, d, bq, bk, k_percent, q8, smooth);
    p.tau = router.tau;
    b200::check(sla2_check_params(&p));
    const std::size_t esz = p.dtype == SLA2_F32 ? 4 : 2;
    b200::DeviceBuffer dq(n * d * esz), dk(n * d * esz), dv(n * d * esz), dout(n * d * esz);
    b200::DeviceBuffer dpq(d * d * 4), dpk(d * d * 4), drho(tm * 4), dmask(tm * tn);
    b200::upload_as(dq, q, p);
    b200::upload_as(dk, k, p);
    b200::upload_as(dv, v, p);
    dpq.upload(router.proj_q.data().data(), d * d * 4);
    dpk.upload(router.proj_k.data().data(), d * d * 4);
    drho.upload(mix.rho.data().data(), tm * 4);
    const size_t ws = sla2_workspace_size(&p);
    b200::DeviceBuffer dws(ws);
    b200::check(sla2_forward(&p, dq.p, dk.p, dv.p, dpq.as<float>(), dpk.as<float>(), drho.as<float>(), dout.p,
                             dmask.as<uint8_t>(), nullptr, nullptr, dws.p, ws, nullptr));
    b200::cuda_check(cudaDeviceSynchronize(), "sla2_attention");
    if (mask_out) {
        *mask_out = BlockMask::zeros(tm, tn);
        mask_out->keep_per_row = topk_budget(k_percent, tn);
        dmask.download(mask_out->bits.data(), tm * tn);
    }
    return b200::download_as(dout, n, d, p);
}

// ------------------------------------------------------------------ RTEN1 files (tensor_io.hpp:12-115)
// magic "RTEN1\0" | u32le rank | u32le dims[rank] | u8 dtype (0 = f32, 1 = f64) | raw LE data.
// The golden-exchange format of the reference's harness; same names, same errors.
namespace rten {
template <class T>
constexpr std::uint8_t dtype_code() {
    static_assert(std::is_same<T, float>::value || std::is_same<T, double>::value, "RTEN1 supports f32 and f64 only");
    return std::is_same<T, float>::value ? 0 : 1;
}
namespace io {
inline void put_u32(std::ostream& os, std::uint32_t v) {
    const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                                (unsigned char)(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
}
inline std::uint32_t get_u32(std::istream& is) {
    unsigned char b[4] = {0, 0, 0, 0};
    is.read(reinterpret_cast<char*>(b), 4);
    return (std::uint32_t)b[0] | ((std::uint32_t)b[1] << 8) | ((std::uint32_t)b[2] << 16) | ((std::uint32_t)b[3] << 24);
}
template <class T>
void write(const std::string& path, const std::vector<std::uint32_t>& dims, const std::vector<T>& data) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw contract_error("RTEN1: cannot open for write: " + path);
    os.write("RTEN1\0", 6);
    put_u32(os, (std::uint32_t)dims.size());
    for (std::uint32_t d : dims) put_u32(os, d);
    const std::uint8_t code = dtype_code<T>();
    os.write(reinterpret_cast<const char*>(&code), 1);
    os.write(reinterpret_cast<const char*>(data.data()), (std::streamsize)(data.size() * sizeof(T)));
}
template <class T>
std::vector<T> read(const std::string& path, std::vector<std::uint32_t>& dims) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw contract_error("RTEN1: cannot open: " + path);
    char magic[6];
    is.read(magic, 6);
    if (!is || std::memcmp(magic, "RTEN1\0", 6) != 0) throw contract_error("RTEN1: bad magic in " + path);
    dims.assign(get_u32(is), 0);
    std::size_t count = 1;
    for (auto& d : dims) count *= (d = get_u32(is));
    std::uint8_t code = 0xff;
    is.read(reinterpret_cast<char*>(&code), 1);
    if (code != dtype_code<T>()) throw contract_error("RTEN1: dtype mismatch in " + path);
    std::vector<T> data(count);
    is.read(reinterpret_cast<char*>(data.data()), (std::streamsize)(count * sizeof(T)));
    if (!is) throw contract_error("RTEN1: truncated file " + path);
    return data;
}
}  // namespace io

template <class T>
void save(const std::string& path, const Matrix<T>& m) {
    io::write(path, {(std::uint32_t)m.rows(), (std::uint32_t)m.cols()}, m.data());
}
template <class T>
void save(const std::string& path, const Vector<T>& v) {
    io::write(path, {(std::uint32_t)v.size()}, v.data());
}
template <class T>
Matrix<T> load_matrix(const std::string& path) {
    std::vector<std::uint32_t> dims;
    std::vector<T> data = io::read<T>(path, dims);
    if (dims.size() != 2) throw contract_error("RTEN1: expected rank 2 in " + path);
    return Matrix<T>(dims[0], dims[1], std::move(data));
}
template <class T>
Vector<T> load_vector(const std::string& path) {
    std::vector<std::uint32_t> dims;
    std::vector<T> data = io::read<T>(path, dims);
    if (dims.size() != 1) throw contract_error("RTEN1: expected rank 1 in " + path);
    return Vector<T>(std::move(data));
}
}  // namespace rten

}  // namespace sla2
