#include <algorithm>
#include <cmath>
// test_shim.cpp -- the reference's own forward-path tests (proj/tests/test_router.cpp,
// test_quant.cpp, test_attention.cpp), re-expressed against the drop-in header
// include/sla2_b200/sla2.hpp, with the CPU oracle (oracle/liboracle.so, TEST INFRASTRUCTURE)
// as the checker. Built and run by tests/test_gpu_shim.py (needs an sm_100a GPU).
#include <cstdio>
#include <functional>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include <cuda_bf16.h>

#include "../../oracle/sla2_oracle.h"
#include "sla2_b200/sla2.hpp"
#ifdef SLA2_B200_MODE_REFERENCE
// built on the reference's own types (oracle/Makefile `dropin`): its RTEN1 I/O and the
// drop-in's composition helper
#include "sla2/tensor_io.hpp"
using sla2::b200::sla2_attention;
#endif

using namespace sla2;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond)                                                                 \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++g_fail;                                                                \
        } else {                                                                     \
            ++g_pass;                                                                \
        }                                                                            \
    } while (0)
template <class E>
static bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Matrix<float> gaussian(std::size_t r, std::size_t c, uint64_t seed, double sd = 1.0) {
    Matrix<float> m(r, c);
    sla2o_gaussian_matrix_f(m.data().data(), m.size(), seed, sd);
    return m;
}
static Matrix<float> uniform(std::size_t r, std::size_t c, uint64_t seed) {
    Matrix<float> m(r, c);
    sla2o_random_matrix_f(m.data().data(), m.size(), seed, -1.0, 1.0);
    return m;
}
static float max_abs_diff(const Matrix<float>& a, const Matrix<float>& b) {
    float m = 0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a.data()[i] - b.data()[i]));
    return m;
}
static float max_abs(const Matrix<float>& a) {
    float m = 0;
    for (float v : a.data()) m = std::max(m, std::fabs(v));
    return m;
}

// test_router.cpp:58-89
static void hard_topk_kats() {
    BlockMask m = hard_topk(Matrix<float>(1, 4, {0.1f, 0.5f, 0.2f, 0.2f}), 25.0);
    EXPECT(m.keep_per_row == 1 && m.at(0, 1) == 1 && m.at(0, 0) == 0 && m.at(0, 2) == 0);
    m = hard_topk(Matrix<float>(1, 4, {0.3f, 0.3f, 0.2f, 0.2f}), 25.0);
    EXPECT(m.at(0, 0) == 1 && m.at(0, 1) == 0);
    Matrix<float> pc = uniform(8, 16, 111);
    m = hard_topk(pc, 25.0);
    std::vector<uint8_t> ref(8 * 16);
    std::size_t kappa = 0;
    sla2o_hard_topk_f(pc.data().data(), 8, 16, 25.0, ref.data(), &kappa);
    EXPECT(m.bits == ref && kappa == 4);
    EXPECT(throws<shape_error>([] { hard_topk(Matrix<float>(1, 4), 0.0); }));
    EXPECT(throws<shape_error>([] { hard_topk(Matrix<float>(1, 4), 101.0); }));
}

// test_router.cpp:12-30 and the router bit-exactness vs the oracle
static void block_scores_tests() {
    Matrix<float> z(16, 4, 0.f);
    Matrix<float> pc = block_scores(z, z, RouterParams<float>::identity(4), 4, 2);
    bool uniform_ok = true;
    for (float v : pc.data()) uniform_ok &= (v == 1.0f / 8.0f);
    EXPECT(uniform_ok);
    const std::size_t n = 512, d = 32, bq = 32, bk = 16;
    Matrix<float> q = gaussian(n, d, 103), k = gaussian(n, d, 104);
    RouterParams<float> rp{gaussian(d, d, 105), gaussian(d, d, 106), 0.1f};
    Matrix<float> got = block_scores(q, k, rp, bq, bk);
    Matrix<float> ref(n / bq, n / bk);
    sla2o_block_scores_f(q.data().data(), k.data().data(), n, d, rp.proj_q.data().data(), rp.proj_k.data().data(),
                         0.1f, bq, bk, ref.data().data());
    EXPECT(got.data() == ref.data());  // bit-exact
    EXPECT(throws<numeric_error>([&] { block_scores(q, k, RouterParams<float>{rp.proj_q, rp.proj_k, 0.f}, bq, bk); }));
}

// quant.hpp:88-96 / test_quant.cpp:87-112
static void smooth_k_tests() {
    Matrix<float> k = gaussian(4096, 64, 209);
    auto [kt, mu] = smooth_k(k);
    std::vector<float> rkt(k.size()), rmu(64);
    sla2o_smooth_k_f(k.data().data(), 4096, 64, rkt.data(), rmu.data());
    EXPECT(kt.data() == rkt && mu.data() == rmu);  // bit-exact serial column mean
    auto [kc, mc] = smooth_k(Matrix<float>(6, 3, 2.5f));
    EXPECT(max_abs(kc) == 0.0f && mc[0] == 2.5f);
}

// test_attention.cpp:215-241, 305-311 through the fp32 path
static void blockwise_tests() {
    for (uint64_t seed : {351u, 352u, 353u}) {
        for (double kp : {10.0, 25.0, 50.0}) {
            const std::size_t n = 64, d = 8, bq = 8, bk = 4;
            AttentionInputs<float> in{gaussian(n, d, seed), gaussian(n, d, seed + 1), gaussian(n, d, seed + 2), bq, bk};
            auto [kt, mu] = smooth_k(in.k);
            BlockMask mask = hard_topk(block_scores(in.q, kt, RouterParams<float>::identity(d), bq, bk), kp);
            MixRatio<float> mix = MixRatio<float>::zeros(in.tm());
            auto [out, saved] = sla2_forward_blockwise(in, Routing<float>{mask}, mix);
            Matrix<float> ref(n, d);
            sla2o_forward_blockwise_f(in.q.data().data(), in.k.data().data(), in.v.data().data(), n, d, bq, bk,
                                      mask.bits.data(), mix.rho.data().data(), 0, 1, ref.data().data(), nullptr, nullptr,
                                      nullptr);
            EXPECT(max_abs_diff(out, ref) <= 1e-4f);
        }
    }
    // empty row -> shape_error; a SoftMask of the wrong geometry -> shape_error (attention.hpp:438-440)
    AttentionInputs<float> in{gaussian(16, 4, 362), gaussian(16, 4, 363), gaussian(16, 4, 364), 4, 4};
    BlockMask mask = BlockMask::zeros(4, 4);
    mask.at(0, 0) = mask.at(1, 1) = mask.at(2, 2) = 1;
    EXPECT(throws<shape_error>([&] { sla2_forward_blockwise(in, Routing<float>{mask}, MixRatio<float>::zeros(4)); }));
    EXPECT(throws<shape_error>(
        [&] { sla2_forward_blockwise(in, Routing<float>{SoftMask<float>{}}, MixRatio<float>::zeros(4)); }));
    // full mask: alpha forced to 1 -> O_s
    auto [o, s] = sla2_forward_blockwise(in, Routing<float>{BlockMask::ones(4, 4)}, MixRatio<float>::constant(4, -5.f));
    EXPECT(max_abs_diff(o, s.o_s) == 0.0f);
}

// the Tape::sla2_attention composition, fp32 (cfg1 blocks) and bf16 (Wan blocks)
static void attention_tests() {
    {
        const std::size_t n = 4096, d = 64, bq = 64, bk = 64;
        Matrix<float> q = gaussian(n, d, 1), k = gaussian(n, d, 2), v = gaussian(n, d, 3);
        RouterParams<float> rp = RouterParams<float>::identity(d);
        MixRatio<float> mix{Vector<float>(n / bq, 0.25f)};
        b200::precision() = b200::Precision::fp32;
        BlockMask mask;
        Matrix<float> out = sla2_attention(q, k, v, mix, rp, bq, bk, 10.0, nullptr, true, &mask);
        Matrix<float> ref(n, d);
        std::vector<uint8_t> rmask((n / bq) * (n / bk));
        sla2o_attention_f(q.data().data(), k.data().data(), v.data().data(), n, d, bq, bk, rp.proj_q.data().data(),
                          rp.proj_k.data().data(), mix.rho.data().data(), 10.0, 0, 1, ref.data().data(), rmask.data(),
                          nullptr, nullptr, nullptr);
        EXPECT(mask.bits == rmask);
        EXPECT(max_abs_diff(out, ref) <= 1e-4f);
    }
    {
        const std::size_t n = 2048, d = 128, bq = 128, bk = 64;
        Matrix<float> q = gaussian(n, d, 4), k = gaussian(n, d, 5), v = gaussian(n, d, 6);
        for (auto* m : {&q, &k, &v})  // the bf16 path sees bf16-valued inputs
            for (float& x : m->data()) x = __bfloat162float(__float2bfloat16_rn(x));
        RouterParams<float> rp = RouterParams<float>::identity(d);
        MixRatio<float> mix{Vector<float>(n / bq, 0.5f)};
        b200::precision() = b200::Precision::bf16;
        BlockMask mask;
        Matrix<float> out = sla2_attention(q, k, v, mix, rp, bq, bk, 5.0, nullptr, true, &mask);
        Matrix<float> ref(n, d);
        std::vector<uint8_t> rmask((n / bq) * (n / bk));
        sla2o_attention_f(q.data().data(), k.data().data(), v.data().data(), n, d, bq, bk, rp.proj_q.data().data(),
                          rp.proj_k.data().data(), mix.rho.data().data(), 5.0, 0, 1, ref.data().data(), rmask.data(),
                          nullptr, nullptr, nullptr);
        EXPECT(mask.bits == rmask);
        EXPECT(max_abs_diff(out, ref) <= 1e-2f * max_abs(ref));
        b200::precision() = b200::Precision::fp32;
    }
}

// RTEN1 (tensor_io.hpp): round trip and the reference's error messages
static void rten_tests() {
    const std::string f = "/tmp/sla2_shim_rten_test.rten";
    Matrix<float> m = gaussian(5, 7, 11);
    rten::save(f, m);
    Matrix<float> back = rten::load_matrix<float>(f);
    EXPECT(back.rows() == 5 && back.cols() == 7 && back.data() == m.data());
    bool threw = false;
    try {
        (void)rten::load_matrix<double>(f);
    } catch (const contract_error& e) {
        threw = std::string(e.what()).find("dtype mismatch") != std::string::npos;
    }
    EXPECT(threw);
    Vector<double> v(std::vector<double>{1.0, -2.5, 3.25});
    rten::save(f, v);
    EXPECT(rten::load_vector<double>(f).data() == v.data());
    threw = false;
    try {
        (void)rten::load_matrix<double>(f);
    } catch (const contract_error& e) {
        threw = std::string(e.what()).find("expected rank 2") != std::string::npos;
    }
    EXPECT(threw);
    std::remove(f.c_str());
}

// sla2_backward (attention.hpp:610-809) through the header: on a full mask alpha is forced to 1,
// so dV = P^T dO with P the row softmax of Q K~^T / sqrt(d) (host restatement, double).
static void backward_tests() {
    const std::size_t n = 128, d = 16, b = 32;
    Matrix<float> q = gaussian(n, d, 21), k = gaussian(n, d, 22), v = gaussian(n, d, 23), dout = gaussian(n, d, 24);
    AttentionInputs<float> in{q, k, v, b, b};
    MixRatio<float> mix{Vector<float>(n / b, 0.3f)};
    BlockMask full = BlockMask::zeros(n / b, n / b);
    for (auto& x : full.bits) x = 1;
    full.keep_per_row = n / b;
    b200::precision() = b200::Precision::fp32;
    auto fwd = sla2_forward_blockwise(in, Routing<float>{full}, mix);
    SLA2Gradients<float> g = sla2_backward(fwd.second, in, mix, dout);
    std::vector<double> mu(d, 0.0);
    for (std::size_t r = 0; r < n; ++r)
        for (std::size_t c = 0; c < d; ++c) mu[c] += k(r, c) / (double)n;
    double worst = 0.0, scale = 0.0;
    std::vector<double> p(n);
    std::vector<double> dv(n * d, 0.0);
    for (std::size_t r = 0; r < n; ++r) {
        double mx = -1e300, s = 0.0;
        for (std::size_t t = 0; t < n; ++t) {
            double acc = 0.0;
            for (std::size_t f = 0; f < d; ++f) acc += (double)q(r, f) * ((double)k(t, f) - mu[f]);
            p[t] = acc / std::sqrt((double)d);
            mx = std::max(mx, p[t]);
        }
        for (std::size_t t = 0; t < n; ++t) s += (p[t] = std::exp(p[t] - mx));
        for (std::size_t t = 0; t < n; ++t)
            for (std::size_t c = 0; c < d; ++c) dv[t * d + c] += p[t] / s * dout(r, c);
    }
    for (std::size_t e = 0; e < n * d; ++e) {
        worst = std::max(worst, std::abs(dv[e] - (double)g.dv.data()[e]));
        scale = std::max(scale, std::abs(dv[e]));
    }
    EXPECT(worst <= 1e-4 * scale);
    bool all_zero = true;
    for (std::size_t i = 0; i < n / b; ++i) all_zero &= g.drho[i] == 0.0f;
    EXPECT(all_zero);  // full rows: alpha forced to 1, no rho gradient (attention.hpp:648-651)
}

// stage-1 soft routing: test_router.cpp:118-165 (soft_topk) and test_attention.cpp:282-292
// (SoftRoutingMatchesNaive) on the device path; the naive side is a host restatement in double.
static void soft_tests() {
    {
        Matrix<float> pc(1, 4, std::vector<float>{0.7f, 0.7f, 0.7f, 0.7f});
        SoftMask<float> sm = soft_topk(pc, 50.0, 0.1f);  // kappa = 2
        for (std::size_t j = 0; j < 4; ++j) EXPECT(std::fabs(sm.values(0, j) - 0.5f) <= 1e-6f);
        EXPECT(sm.budget == 2);
    }
    {
        Matrix<float> pc = uniform(6, 12, 122);
        SoftMask<float> sm = soft_topk(pc, 25.0, 0.1f);  // kappa = 3
        for (std::size_t i = 0; i < 6; ++i) {
            double s = 0;
            for (std::size_t j = 0; j < 12; ++j) s += sm.values(i, j);
            EXPECT(std::fabs(s - 3.0) <= 1e-5);
        }
        EXPECT(throws<numeric_error>([&] { soft_topk(pc, 25.0, 0.0f); }));
        // soft_topk_backward (test_router.cpp:173-178): zero upstream -> zero; the diagonal rule
        Matrix<float> zero(6, 12, 0.0f);
        Matrix<float> g0 = soft_topk_backward(pc, sm, zero);
        EXPECT(max_abs(g0) == 0.0f);
        Matrix<float> up = uniform(6, 12, 134);
        Matrix<float> g = soft_topk_backward(pc, sm, up);
        float worst = 0.0f;
        for (std::size_t e = 0; e < pc.size(); ++e) {
            const float v = sm.values.data()[e];
            worst = std::max(worst, std::fabs(g.data()[e] - up.data()[e] * v * (1.0f - v) * (1.0f / 0.1f)));
        }
        EXPECT(worst == 0.0f);
    }
    const std::size_t n = 32, d = 8, bq = 4, bk = 4, tm = n / bq, tn = n / bk;
    AttentionInputs<float> in{gaussian(n, d, 359), gaussian(n, d, 360), gaussian(n, d, 361), bq, bk};
    auto [kt, mu] = smooth_k(in.k);
    SoftMask<float> soft = soft_topk(block_scores(in.q, kt, RouterParams<float>::identity(d), bq, bk), 25.0, 0.1f);
    MixRatio<float> mix = MixRatio<float>::constant(tm, 0.3f);
    auto [out, saved] = sla2_forward_blockwise(in, Routing<float>{soft}, mix);
    // naive: sparse = softmax weighted by w over all keys; linear = phi(Q) phi(K~)^T weighted by 1 - w
    std::vector<double> ktd(n * d), pk(n * d);
    for (std::size_t c = 0; c < d; ++c) {
        float acc = 0.0f;
        for (std::size_t r = 0; r < n; ++r) acc += in.k(r, c);
        const float m = acc / (float)n;
        for (std::size_t r = 0; r < n; ++r) ktd[r * d + c] = (double)(in.k(r, c) - m);
    }
    auto softmax_row = [&](const double* x, double* y) {
        double mx = x[0], s = 0;
        for (std::size_t f = 1; f < d; ++f) mx = std::max(mx, x[f]);
        for (std::size_t f = 0; f < d; ++f) s += (y[f] = std::exp(x[f] - mx));
        for (std::size_t f = 0; f < d; ++f) y[f] /= s;
    };
    for (std::size_t r = 0; r < n; ++r) softmax_row(&ktd[r * d], &pk[r * d]);
    double worst = 0;
    for (std::size_t r = 0; r < n; ++r) {
        std::vector<double> qr(d), pq(d), os(d, 0), ol(d, 0);
        for (std::size_t f = 0; f < d; ++f) qr[f] = in.q(r, f);
        softmax_row(qr.data(), pq.data());
        std::vector<double> s(n);
        double mx = -1e300;
        for (std::size_t t = 0; t < n; ++t) {
            double a = 0;
            for (std::size_t f = 0; f < d; ++f) a += qr[f] * ktd[t * d + f];
            s[t] = a / std::sqrt((double)d);
            mx = std::max(mx, s[t]);
        }
        double zs = 0, zl = 0;
        for (std::size_t t = 0; t < n; ++t) {
            const double w = soft.values(r / bq, t / bk);
            const double es = w * std::exp(s[t] - mx);
            double al = 0;
            for (std::size_t f = 0; f < d; ++f) al += pq[f] * pk[t * d + f];
            al *= 1.0 - w;
            zs += es;
            zl += al;
            for (std::size_t c = 0; c < d; ++c) {
                os[c] += es * in.v(t, c);
                ol[c] += al * in.v(t, c);
            }
        }
        const double a = 1.0 / (1.0 + std::exp(-0.3));
        for (std::size_t c = 0; c < d; ++c)
            worst = std::max(worst, std::fabs(out(r, c) - (a * os[c] / zs + (1 - a) * ol[c] / zl)));
    }
    EXPECT(worst <= 1e-5);
    EXPECT(saved.o_s.rows() == n && !saved.hard());
    EXPECT(throws<contract_error>([&] {
        QuantConfig qc;
        sla2_forward_blockwise(in, Routing<float>{soft}, mix, &qc);
    }));
}

int main() {
    rten_tests();
    backward_tests();
    hard_topk_kats();
    block_scores_tests();
    smooth_k_tests();
    blockwise_tests();
    attention_tests();
    soft_tests();
    std::printf("shim tests: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
