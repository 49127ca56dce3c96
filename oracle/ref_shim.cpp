// ref_shim.cpp -- extern "C" bindings over the UNMODIFIED reference headers
// (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against /root/reference/proj/include (and the reference's
// tests/test_util.hpp for its random generators) into oracle/_ref/libsla2_ref.so, which is
// git-ignored. It is the ground truth that pins the C restatement in sla2_oracle.c
// (tests/test_oracle.py compares the two bit for bit) and, when present, the CPU baseline
// arm of bench.py ("kind": "reference"). No reference source is copied here: every call
// goes into the reference's own templates.
#include <cstring>
#include <exception>
#include <vector>

#include "sla2/attention.hpp"
#include "sla2/quant.hpp"
#include "sla2/router.hpp"
#include "sla2/tensor_io.hpp"
#include "test_util.hpp"

using namespace sla2;

namespace {

template <class T>
Matrix<T> wrap(const T* p, std::size_t r, std::size_t c) {
    return Matrix<T>(r, c, std::vector<T>(p, p + r * c));
}

template <class T>
void copy_out(const Matrix<T>& m, T* dst) {
    if (dst) std::memcpy(dst, m.data().data(), sizeof(T) * m.size());
}

int classify(const std::exception& e) {
    if (dynamic_cast<const shape_error*>(&e)) return 1;
    if (dynamic_cast<const numeric_error*>(&e)) return 2;
    if (dynamic_cast<const contract_error*>(&e)) return 3;
    return 9;
}

BlockMask wrap_mask(const std::uint8_t* m, std::size_t tm, std::size_t tn) {
    BlockMask b = BlockMask::zeros(tm, tn);
    std::memcpy(b.bits.data(), m, tm * tn);
    return b;
}

template <class T>
int colmean_(const T* x, std::size_t r, std::size_t c, T* out) {
    try {
        auto v = colmean(wrap(x, r, c));
        std::memcpy(out, v.data().data(), sizeof(T) * c);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int smooth_k_(const T* k, std::size_t r, std::size_t c, T* kt, T* mean) {
    try {
        auto [m, mu] = smooth_k(wrap(k, r, c));
        copy_out(m, kt);
        std::memcpy(mean, mu.data().data(), sizeof(T) * c);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int block_scores_(const T* q, const T* k, std::size_t n, std::size_t d, const T* pq, const T* pk,
                  T tau, std::size_t bq, std::size_t bk, T* pc) {
    try {
        RouterParams<T> rp{wrap(pq, d, d), wrap(pk, d, d), tau};
        copy_out(block_scores(wrap(q, n, d), wrap(k, n, d), rp, bq, bk), pc);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int hard_topk_(const T* pc, std::size_t tm, std::size_t tn, double kp, std::uint8_t* mask,
               std::size_t* kappa) {
    try {
        BlockMask m = hard_topk(wrap(pc, tm, tn), kp);
        std::memcpy(mask, m.bits.data(), tm * tn);
        if (kappa) *kappa = m.keep_per_row;
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int quantize_(const T* x, std::size_t n, std::int8_t* codes, T* scale) {
    try {
        auto qb = quantize(wrap(x, 1, n));
        std::memcpy(codes, qb.values.data(), n);
        *scale = qb.scale;
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int forward_blockwise_(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,
                       std::size_t bq, std::size_t bk, const std::uint8_t* mask, const T* rho,
                       int quant, int smooth, T* out, T* o_s, T* o_l, T* big_l) {
    try {
        AttentionInputs<T> in{wrap(q, n, d), wrap(k, n, d), wrap(v, n, d), bq, bk};
        MixRatio<T> mix{Vector<T>(std::vector<T>(rho, rho + n / bq))};
        QuantConfig qc;
        auto [o, saved] = sla2_forward_blockwise(in, Routing<T>{wrap_mask(mask, n / bq, n / bk)},
                                                 mix, quant ? &qc : nullptr, smooth != 0);
        copy_out(o, out);
        copy_out(saved.o_s, o_s);
        copy_out(saved.o_l, o_l);
        if (big_l) std::memcpy(big_l, saved.big_l.data().data(), sizeof(T) * n);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// sla2_forward_blockwise's full SLA2ForwardSaved (attention.hpp:345-358): h_blocks [tm][d][d],
// z_blocks [tm][d], q_phi / k_phi [n][d] besides o_s, o_l, big_l.
template <class T>
int forward_saved_(const T* q, const T* k, const T* v, std::size_t n, std::size_t d, std::size_t bq,
                   std::size_t bk, const std::uint8_t* mask, const T* rho, int quant, int smooth, T* out, T* o_s,
                   T* o_l, T* big_l, T* h_blocks, T* z_blocks, T* q_phi, T* k_phi) {
    try {
        AttentionInputs<T> in{wrap(q, n, d), wrap(k, n, d), wrap(v, n, d), bq, bk};
        MixRatio<T> mix{Vector<T>(std::vector<T>(rho, rho + n / bq))};
        QuantConfig qc;
        auto [o, saved] = sla2_forward_blockwise(in, Routing<T>{wrap_mask(mask, n / bq, n / bk)}, mix,
                                                 quant ? &qc : nullptr, smooth != 0);
        copy_out(o, out);
        copy_out(saved.o_s, o_s);
        copy_out(saved.o_l, o_l);
        std::memcpy(big_l, saved.big_l.data().data(), sizeof(T) * n);
        for (std::size_t i = 0; i < saved.h_blocks.size(); ++i) {
            copy_out(saved.h_blocks[i], h_blocks + i * d * d);
            std::memcpy(z_blocks + i * d, saved.z_blocks[i].data().data(), sizeof(T) * d);
        }
        copy_out(saved.q_phi, q_phi);
        copy_out(saved.k_phi, k_phi);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// detail::block_scores_qk (attention.hpp:372-394) for one (query block, key block): S = Q_i K_j^T /
// sqrt(d), or through quantize -> quantized_product -> scale when quant (the QAT scores).
template <class T>
int block_scores_qk_(const T* q, const T* k, std::size_t n, std::size_t d, std::size_t qi0, std::size_t bq,
                     std::size_t kj0, std::size_t bk, int quant, T* s) {
    try {
        QuantConfig qc;
        copy_out(detail::block_scores_qk(wrap(q, n, d), wrap(k, n, d), qi0, bq, kj0, bk, quant ? &qc : nullptr), s);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int forward_naive_(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,
                   std::size_t bq, std::size_t bk, const std::uint8_t* mask, const T* rho,
                   int smooth, T* out, T* o_s, T* o_l) {
    try {
        AttentionInputs<T> in{wrap(q, n, d), wrap(k, n, d), wrap(v, n, d), bq, bk};
        MixRatio<T> mix{Vector<T>(std::vector<T>(rho, rho + n / bq))};
        NaiveDetail<T> det;
        auto o = sla2_forward_naive(in, Routing<T>{wrap_mask(mask, n / bq, n / bk)}, mix,
                                    smooth != 0, &det);
        copy_out(o, out);
        copy_out(det.o_s, o_s);
        copy_out(det.o_l, o_l);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// Tape::sla2_attention's forward composition (tape.hpp:263-272), element type T.
template <class T>
int attention_(const T* q, const T* k, const T* v, std::size_t n, std::size_t d, std::size_t bq,
               std::size_t bk, const T* pq, const T* pk, const T* rho, double kp, int quant,
               int smooth, T* out, std::uint8_t* mask_out, T* o_s, T* o_l, T* big_l) {
    try {
        AttentionInputs<T> in{wrap(q, n, d), wrap(k, n, d), wrap(v, n, d), bq, bk};
        MixRatio<T> mix{Vector<T>(std::vector<T>(rho, rho + n / bq))};
        RouterParams<T> rp{wrap(pq, d, d), wrap(pk, d, d), T(0.1)};
        Matrix<T> kt = smooth ? smooth_k(in.k).first : in.k;
        BlockMask mask = hard_topk(block_scores(in.q, kt, rp, bq, bk), kp);
        QuantConfig qc;
        auto [o, saved] = sla2_forward_blockwise(in, Routing<T>{mask}, mix,
                                                 quant ? &qc : nullptr, smooth != 0);
        copy_out(o, out);
        if (mask_out) std::memcpy(mask_out, mask.bits.data(), mask.bits.size());
        copy_out(saved.o_s, o_s);
        copy_out(saved.o_l, o_l);
        if (big_l) std::memcpy(big_l, saved.big_l.data().data(), sizeof(T) * n);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

template <class T>
int backward_(const T* q, const T* k, const T* v, std::size_t n, std::size_t d, std::size_t bq, std::size_t bk,
              const std::uint8_t* mask, const T* rho, int smooth, const T* d_out, T* dq, T* dk, T* dv, T* drho,
              T* o_s, T* o_l, T* big_l) {
    try {
        AttentionInputs<T> in{wrap(q, n, d), wrap(k, n, d), wrap(v, n, d), bq, bk};
        MixRatio<T> mix{Vector<T>(std::vector<T>(rho, rho + n / bq))};
        Routing<T> routing{wrap_mask(mask, n / bq, n / bk)};
        auto fwd = sla2_forward_blockwise(in, routing, mix, nullptr, smooth != 0);
        const SLA2ForwardSaved<T>& saved = fwd.second;
        SLA2Gradients<T> g = sla2_backward(saved, in, mix, wrap(d_out, n, d));
        copy_out(g.dq, dq);
        copy_out(g.dk, dk);
        copy_out(g.dv, dv);
        std::memcpy(drho, g.drho.data().data(), sizeof(T) * (n / bq));
        copy_out(saved.o_s, o_s);
        copy_out(saved.o_l, o_l);
        if (big_l) std::memcpy(big_l, saved.big_l.data().data(), sizeof(T) * n);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// soft_topk (router.hpp:126-190): values and lambdas of one [tm, tn] score matrix
template <class T>
int soft_topk_(const T* pc, std::size_t tm, std::size_t tn, double kp, T tau, T* values, T* lambdas) {
    try {
        SoftMask<T> sm = soft_topk(wrap(pc, tm, tn), kp, tau);
        copy_out(sm.values, values);
        std::memcpy(lambdas, sm.lambdas.data().data(), sizeof(T) * tm);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// soft_topk_backward (router.hpp:197-212) on the reference's own SoftMask from soft_topk
template <class T>
int soft_topk_backward_(const T* pc, std::size_t tm, std::size_t tn, double kp, T tau, const T* upstream, T* grad) {
    try {
        SoftMask<T> sm = soft_topk(wrap(pc, tm, tn), kp, tau);
        copy_out(soft_topk_backward(wrap(pc, tm, tn), sm, wrap(upstream, tm, tn)), grad);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// sla2_forward_blockwise with Routing = SoftMask (attention.hpp:484-558), caller-given values
template <class T>
int forward_soft_(const T* q, const T* k, const T* v, std::size_t n, std::size_t d, std::size_t bq,
                  std::size_t bk, const T* values, const T* rho, int smooth, T* out, T* o_s, T* o_l,
                  T* big_l) {
    try {
        AttentionInputs<T> in{wrap(q, n, d), wrap(k, n, d), wrap(v, n, d), bq, bk};
        MixRatio<T> mix{Vector<T>(std::vector<T>(rho, rho + n / bq))};
        SoftMask<T> sm;
        sm.tm = n / bq;
        sm.tn = n / bk;
        sm.values = wrap(values, sm.tm, sm.tn);
        sm.lambdas = Vector<T>(sm.tm);
        auto [o, saved] = sla2_forward_blockwise(in, Routing<T>{sm}, mix, nullptr, smooth != 0);
        copy_out(o, out);
        copy_out(saved.o_s, o_s);
        copy_out(saved.o_l, o_l);
        if (big_l) std::memcpy(big_l, saved.big_l.data().data(), sizeof(T) * n);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

}  // namespace

extern "C" {

#define SLA2R_INST(T, S)                                                                          \
    int sla2r_colmean_##S(const T* x, std::size_t r, std::size_t c, T* out) {                    \
        return colmean_<T>(x, r, c, out);                                                         \
    }                                                                                             \
    int sla2r_smooth_k_##S(const T* k, std::size_t r, std::size_t c, T* kt, T* mean) {           \
        return smooth_k_<T>(k, r, c, kt, mean);                                                   \
    }                                                                                             \
    int sla2r_block_scores_##S(const T* q, const T* k, std::size_t n, std::size_t d, const T* pq, \
                               const T* pk, T tau, std::size_t bq, std::size_t bk, T* pc) {      \
        return block_scores_<T>(q, k, n, d, pq, pk, tau, bq, bk, pc);                             \
    }                                                                                             \
    int sla2r_hard_topk_##S(const T* pc, std::size_t tm, std::size_t tn, double kp,             \
                            std::uint8_t* mask, std::size_t* kappa) {                            \
        return hard_topk_<T>(pc, tm, tn, kp, mask, kappa);                                        \
    }                                                                                             \
    int sla2r_quantize_##S(const T* x, std::size_t n, std::int8_t* codes, T* scale) {            \
        return quantize_<T>(x, n, codes, scale);                                                  \
    }                                                                                             \
    int sla2r_forward_blockwise_##S(const T* q, const T* k, const T* v, std::size_t n,           \
                                    std::size_t d, std::size_t bq, std::size_t bk,               \
                                    const std::uint8_t* mask, const T* rho, int quant,           \
                                    int smooth, T* out, T* o_s, T* o_l, T* big_l) {              \
        return forward_blockwise_<T>(q, k, v, n, d, bq, bk, mask, rho, quant, smooth, out, o_s,  \
                                     o_l, big_l);                                                 \
    }                                                                                             \
    int sla2r_forward_saved_##S(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,  \
                                std::size_t bq, std::size_t bk, const std::uint8_t* mask,        \
                                const T* rho, int quant, int smooth, T* out, T* o_s, T* o_l,     \
                                T* big_l, T* hb, T* zb, T* qp, T* kp) {                          \
        return forward_saved_<T>(q, k, v, n, d, bq, bk, mask, rho, quant, smooth, out, o_s, o_l, \
                                 big_l, hb, zb, qp, kp);                                         \
    }                                                                                             \
    int sla2r_block_scores_qk_##S(const T* q, const T* k, std::size_t n, std::size_t d,         \
                                  std::size_t qi0, std::size_t bq, std::size_t kj0, std::size_t bk, \
                                  int quant, T* s) {                                             \
        return block_scores_qk_<T>(q, k, n, d, qi0, bq, kj0, bk, quant, s);                      \
    }                                                                                             \
    int sla2r_forward_naive_##S(const T* q, const T* k, const T* v, std::size_t n, std::size_t d, \
                                std::size_t bq, std::size_t bk, const std::uint8_t* mask,        \
                                const T* rho, int smooth, T* out, T* o_s, T* o_l) {              \
        return forward_naive_<T>(q, k, v, n, d, bq, bk, mask, rho, smooth, out, o_s, o_l);       \
    }                                                                                             \
    int sla2r_attention_##S(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,    \
                            std::size_t bq, std::size_t bk, const T* pq, const T* pk,            \
                            const T* rho, double kp, int quant, int smooth, T* out,              \
                            std::uint8_t* mask, T* o_s, T* o_l, T* big_l) {                      \
        return attention_<T>(q, k, v, n, d, bq, bk, pq, pk, rho, kp, quant, smooth, out, mask,   \
                             o_s, o_l, big_l);                                                    \
    }                                                                                             \
    void sla2r_gaussian_matrix_##S(T* out, std::size_t n, std::uint64_t seed, double sd) {       \
        auto m = testutil::gaussian_matrix<T>(1, n, seed, T(sd));                                 \
        std::memcpy(out, m.data().data(), sizeof(T) * n);                                         \
    }                                                                                             \
    void sla2r_random_matrix_##S(T* out, std::size_t n, std::uint64_t seed, double lo,           \
                                 double hi) {                                                     \
        auto m = testutil::random_matrix<T>(1, n, seed, T(lo), T(hi));                            \
        std::memcpy(out, m.data().data(), sizeof(T) * n);                                         \
    }

SLA2R_INST(float, f)
SLA2R_INST(double, d)

// attention.hpp:610-809 on the reference's own forward state (sla2_forward_blockwise, hard mask)
#define SLA2R_BWD(T, S)                                                                           \
    int sla2r_backward_##S(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,     \
                           std::size_t bq, std::size_t bk, const std::uint8_t* mask, const T* rho, \
                           int smooth, const T* d_out, T* dq, T* dk, T* dv, T* drho, T* o_s,      \
                           T* o_l, T* big_l) {                                                   \
        return backward_<T>(q, k, v, n, d, bq, bk, mask, rho, smooth, d_out, dq, dk, dv, drho, o_s, \
                            o_l, big_l);                                                          \
    }
SLA2R_BWD(float, f)
SLA2R_BWD(double, d)

// RTEN1 through the reference's own sla2::rten (tensor_io.hpp): rank-2 save / load (rank 1 when
// rows == 0), so the exchange format is checked against the reference's writer and reader.
#define SLA2R_RTEN(T, S)                                                                          \
    int sla2r_rten_save_##S(const char* path, std::size_t rows, std::size_t cols, const T* data) { \
        try {                                                                                     \
            if (rows == 0) rten::save(path, Vector<T>(std::vector<T>(data, data + cols)));        \
            else rten::save(path, wrap(data, rows, cols));                                        \
            return 0;                                                                             \
        } catch (const std::exception& e) { return classify(e); }                                 \
    }                                                                                             \
    int sla2r_rten_load_##S(const char* path, std::size_t rows, std::size_t cols, T* out) {      \
        try {                                                                                     \
            if (rows == 0) {                                                                      \
                auto v = rten::load_vector<T>(path);                                              \
                if (v.size() != cols) return 1;                                                   \
                std::memcpy(out, v.data().data(), sizeof(T) * cols);                              \
            } else {                                                                              \
                auto m = rten::load_matrix<T>(path);                                              \
                if (m.rows() != rows || m.cols() != cols) return 1;                               \
                copy_out(m, out);                                                                 \
            }                                                                                     \
            return 0;                                                                             \
        } catch (const std::exception& e) { return classify(e); }                                 \
    }
SLA2R_RTEN(float, f)
SLA2R_RTEN(double, d)

#define SLA2R_SOFT(T, S)                                                                          \
    int sla2r_soft_topk_##S(const T* pc, std::size_t tm, std::size_t tn, double kp, T tau, T* values, \
                            T* lambdas) {                                                         \
        return soft_topk_<T>(pc, tm, tn, kp, tau, values, lambdas);                               \
    }                                                                                             \
    int sla2r_soft_topk_backward_##S(const T* pc, std::size_t tm, std::size_t tn, double kp, T tau,          \
                                     const T* upstream, T* grad) {                                \
        return soft_topk_backward_<T>(pc, tm, tn, kp, tau, upstream, grad);                       \
    }                                                                                             \
    int sla2r_forward_soft_##S(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,  \
                               std::size_t bq, std::size_t bk, const T* values, const T* rho,     \
                               int smooth, T* out, T* o_s, T* o_l, T* big_l) {                    \
        return forward_soft_<T>(q, k, v, n, d, bq, bk, values, rho, smooth, out, o_s, o_l, big_l); \
    }
SLA2R_SOFT(float, f)
SLA2R_SOFT(double, d)

std::size_t sla2r_topk_budget(double kp, std::size_t tn) { return topk_budget(kp, tn); }
std::size_t sla2r_max_worker_threads(void) { return max_worker_threads(); }

}  // extern "C"
