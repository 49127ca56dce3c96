// model_dropin.cpp -- one step of the reference's toy DiT (model.hpp) with SLA2 attention in
// every head, TEST INFRASTRUCTURE. Built twice from the UNMODIFIED reference headers by
// oracle/Makefile (`make -C oracle dropin`, only where /root/reference exists; the binaries
// travel to the GPU box in oracle/_ref/):
//   model_ref   the reference as is (CPU)
//   model_b200  the same source with -DSLA2_B200_DROPIN: include/sla2_b200/sla2.hpp comes first,
//               so Tape::sla2_attention (tape.hpp:263-286) -> smooth_k / block_scores /
//               hard_topk / sla2_forward_blockwise run on the B200 through the C ABI, and the
//               reference's own sla2_backward consumes the drop-in's SLA2ForwardSaved.
// Each writes: [u32 count][f64 values] blocks -- model output (n x d_model), the loss, dL/dw_in,
// dL/dwq of layer 0, and every head's router mask (as 0/1 doubles).
#ifdef SLA2_B200_DROPIN
#include "sla2_b200/sla2.hpp"
#ifndef SLA2_B200_MODE_REFERENCE
#error "the drop-in must build on the reference's own types here"
#endif
#endif
#include <cstdio>
#include <random>
#include <vector>

#include "sla2/model.hpp"
#include "sla2/tape.hpp"

static void put(FILE* f, const std::vector<double>& v) {
    const unsigned n = (unsigned)v.size();
    fwrite(&n, 4, 1, f);
    fwrite(v.data(), 8, v.size(), f);
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s out.bin [k_percent] [seed]\n", argv[0]);
        return 2;
    }
    const double kp = argc > 2 ? std::atof(argv[2]) : 25.0;
    const unsigned seed = argc > 3 ? (unsigned)std::atoi(argv[3]) : 7;
    try {
        sla2::ModelConfig cfg;  // n = 256, d_model = 64, 2 heads (d = 32), 2 layers, bq = 16, bk = 8
        const sla2::ToyModelParams p = sla2::init_toy_model(cfg, seed);
        sla2::ad::Tape tape;
        const sla2::ModelVars mv = sla2::register_model(tape, p);
        std::mt19937_64 rng(seed + 100);
        std::normal_distribution<double> nd(0.0, 1.0);
        sla2::Matrix<double> x(cfg.n, cfg.d_model);
        for (auto& e : x.data()) e = nd(rng);
        sla2::AttentionRunOptions opts;
        opts.use_sla2 = true;
        opts.k_percent = kp;
        std::vector<sla2::QKVRecord> cap;
        auto out = sla2::model_forward(tape, p, mv, x, 5, opts, &cap);
        auto loss = tape.mse_against(out, sla2::Matrix<double>(cfg.n, cfg.d_model, 0.0));
        tape.backward(loss);
        FILE* f = std::fopen(argv[1], "wb");
        if (!f) return 3;
        put(f, tape.value(out).data());
        put(f, tape.value(loss).data());
        put(f, tape.grad(mv.w_in).data());
        put(f, tape.grad(mv.layers[0].wq).data());
        for (const auto& r : cap) {  // the router of every (layer, head), as Tape::sla2_attention runs it
            const auto kt = sla2::smooth_k(r.k).first;
            const auto m = sla2::hard_topk(sla2::block_scores(r.q, kt, p.layers[r.layer].router[r.head], cfg.bq, cfg.bk),
                                           kp);
            put(f, std::vector<double>(m.bits.begin(), m.bits.end()));
        }
        std::fclose(f);
        std::printf("ok heads=%zu\n", cap.size());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
