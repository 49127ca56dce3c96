/*
 * sla2_oracle.h -- CPU restatement of the SLA2 forward hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle, not product code. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product path
 * (libsla2_b200.so) never links or calls anything in oracle/.
 *
 * It restates, in plain C, the arithmetic of the reference's header-only library
 * /root/reference/proj/include/sla2/*.hpp for element type float (suffix _f) and double
 * (suffix _d), operation by operation and in the same serial order, so that with
 * `-O2 -ffp-contract=off` (no -march=native, no -ffast-math) its results are
 * bit-identical to the reference built the same way. Every function cites the
 * reference file:line it follows. Parity of this restatement against the unmodified
 * reference is pinned by tests/test_oracle.py (bit-exact vs oracle/_ref built from the
 * reference headers, plus the reference's own known-answer tests re-expressed).
 *
 * Layout: every matrix is row-major, rows x cols, like sla2::Matrix (matrix.hpp:18-23).
 * Errors: functions return 0 on success, or the sla2 error class the reference would
 * throw: 1 = shape_error, 2 = numeric_error, 3 = contract_error (common.hpp:13-29).
 */
#ifndef SLA2_ORACLE_H
#define SLA2_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLA2O_OK 0
#define SLA2O_SHAPE 1
#define SLA2O_NUMERIC 2
#define SLA2O_CONTRACT 3

/* ---- libstdc++-compatible random streams (tests/test_util.hpp:11-36) ---- */
typedef struct { uint64_t mt[312]; int mti; int has_saved; double saved; } sla2o_rng;
void sla2o_rng_seed(sla2o_rng* r, uint64_t seed);            /* std::mt19937_64(seed) */
uint64_t sla2o_rng_next(sla2o_rng* r);                        /* operator() */
double sla2o_rng_canonical(sla2o_rng* r);                     /* generate_canonical<double,53> */
double sla2o_rng_uniform(sla2o_rng* r, double lo, double hi); /* uniform_real_distribution<double> */
double sla2o_rng_normal(sla2o_rng* r, double mean, double sd);/* normal_distribution<double> */
/* testutil::random_matrix / gaussian_matrix: fill rows*cols values cast to T. */
void sla2o_random_matrix_f(float* out, size_t n, uint64_t seed, double lo, double hi);
void sla2o_random_matrix_d(double* out, size_t n, uint64_t seed, double lo, double hi);
void sla2o_gaussian_matrix_f(float* out, size_t n, uint64_t seed, double sd);
void sla2o_gaussian_matrix_d(double* out, size_t n, uint64_t seed, double sd);

/* ---- router.hpp:36-40 ---- */
size_t sla2o_topk_budget(double k_percent, size_t tn);

#define SLA2O_DECLARE(T, S)                                                                      \
    void sla2o_colmean_##S(const T* x, size_t rows, size_t cols, T* out);                        \
    void sla2o_smooth_k_##S(const T* k, size_t rows, size_t cols, T* ktilde, T* mean);           \
    int sla2o_mean_pool_##S(const T* x, size_t rows, size_t cols, size_t block, T* out);         \
    int sla2o_matmul_##S(const T* a, size_t ar, size_t ac, const T* b, size_t br, size_t bc,     \
                         int transpose_b, T* out);                                               \
    void sla2o_row_softmax_##S(const T* s, size_t rows, size_t cols, T* out);                    \
    void sla2o_scale_##S(const T* a, size_t n, T s, T* out);                                     \
    int sla2o_block_scores_##S(const T* q, const T* k, size_t n, size_t d, const T* proj_q,      \
                               const T* proj_k, T tau, size_t bq, size_t bk, T* pc);             \
    int sla2o_hard_topk_##S(const T* pc, size_t tm, size_t tn, double k_percent,                 \
                            uint8_t* mask, size_t* kappa_out);                                   \
    int sla2o_quantize_##S(const T* x, size_t n, int8_t* codes, T* scale);                       \
    int sla2o_quantized_product_##S(const int8_t* a, size_t ar, size_t ac, T sa,                 \
                                    const int8_t* b, size_t br, size_t bc, T sb,                 \
                                    int transpose_b, T* out);                                    \
    T sla2o_sigmoid_##S(T x);                                                                    \
    int sla2o_forward_blockwise_##S(const T* q, const T* k, const T* v, size_t n, size_t d,      \
                                    size_t bq, size_t bk, const uint8_t* mask, const T* rho,     \
                                    int quant, int smooth, T* out, T* o_s, T* o_l, T* big_l);    \
    int sla2o_forward_naive_##S(const T* q, const T* k, const T* v, size_t n, size_t d,          \
                                size_t bq, size_t bk, const uint8_t* mask, const T* rho,         \
                                int smooth, T* out, T* o_s, T* o_l);                             \
    int sla2o_full_attention_##S(const T* q, const T* k, const T* v, size_t n, size_t d,         \
                                 T* out);                                                        \
    int sla2o_attention_##S(const T* q, const T* k, const T* v, size_t n, size_t d, size_t bq,   \
                            size_t bk, const T* proj_q, const T* proj_k, const T* rho,           \
                            double k_percent, int quant, int smooth, T* out, uint8_t* mask,      \
                            T* o_s, T* o_l, T* big_l);                                   \
    /* RAGGED EXTENSION: n need not be divisible by bq / bk; the last   \
     * query / key block is partial. Equal to the functions above when the blocks divide n. */ \
    int sla2o_mean_pool_ragged_##S(const T* x, size_t rows, size_t cols, size_t block, T* out); \
    int sla2o_block_scores_ragged_##S(const T* q, const T* k, size_t n, size_t d,               \
                                      const T* proj_q, const T* proj_k, T tau, size_t bq,       \
                                      size_t bk, T* pc);                                        \
    int sla2o_forward_blockwise_ragged_##S(const T* q, const T* k, const T* v, size_t n,        \
                                           size_t d, size_t bq, size_t bk, const uint8_t* mask, \
                                           const T* rho, int quant, int smooth, T* out, T* o_s, \
                                           T* o_l, T* big_l);                                   \
    int sla2o_attention_ragged_##S(const T* q, const T* k, const T* v, size_t n, size_t d,      \
                                   size_t bq, size_t bk, const T* proj_q, const T* proj_k,      \
                                   const T* rho, double k_percent, int quant, int smooth,       \
                                   T* out, uint8_t* mask, T* o_s, T* o_l, T* big_l);

SLA2O_DECLARE(float, f)
SLA2O_DECLARE(double, d)

/* Worker threads used by sla2o_forward_blockwise_* (over query blocks, like the
 * reference's parallel_for, common.hpp:45-69). Results do not depend on it. */
void sla2o_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
