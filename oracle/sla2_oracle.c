/*
 * sla2_oracle.c -- CPU restatement of the SLA2 forward hot path (TEST INFRASTRUCTURE ONLY).
 * See sla2_oracle.h. Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared -pthread -lm
 * (oracle/Makefile). Never linked into the product library.
 */
#include "sla2_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static int g_oracle_threads = 1;
void sla2o_set_threads(int n) { g_oracle_threads = n < 1 ? 1 : n; }
static int oracle_threads(void) { return g_oracle_threads; }

/* router.hpp:36-40: kappa = min(tn, max(1.0, llround(k%/100 * tn) * 1.0)). */
size_t sla2o_topk_budget(double k_percent, size_t tn) {
    const double r = (double)llround(k_percent / 100.0 * (double)tn) * 1.0;
    const size_t kappa = (size_t)(r > 1.0 ? r : 1.0);
    return kappa < tn ? kappa : tn;
}

/* ---- std::mt19937_64 (the standard's reference engine; used by test_util.hpp:14,24) ---- */
#define MT_N 312
#define MT_M 156
void sla2o_rng_seed(sla2o_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->has_saved = 0;
    r->saved = 0.0;
}

uint64_t sla2o_rng_next(sla2o_rng* r) {
    static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->mti >= MT_N) {
        int i;
        for (i = 0; i < MT_N - MT_M; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ mag[x & 1ULL];
        }
        for (; i < MT_N - 1; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag[x & 1ULL];
        }
        uint64_t x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ mag[x & 1ULL];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* libstdc++ generate_canonical<double, 53>(mt19937_64): one draw, double(x) / 2^64,
 * clamped below 1 by nextafter. */
double sla2o_rng_canonical(sla2o_rng* r) {
    const double sum = (double)sla2o_rng_next(r);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* libstdc++ uniform_real_distribution<double>: canonical * (b - a) + a. */
double sla2o_rng_uniform(sla2o_rng* r, double lo, double hi) {
    return sla2o_rng_canonical(r) * (hi - lo) + lo;
}

/* libstdc++ normal_distribution<double>: Marsaglia polar method with one cached value. */
double sla2o_rng_normal(sla2o_rng* r, double mean, double sd) {
    double ret;
    if (r->has_saved) {
        r->has_saved = 0;
        ret = r->saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * sla2o_rng_canonical(r) - 1.0;
            y = 2.0 * sla2o_rng_canonical(r) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(-2 * log(r2) / r2);
        r->saved = x * mult;
        r->has_saved = 1;
        ret = y * mult;
    }
    return ret * sd + mean;
}

/* float instantiation (Matrix<float>): accumulator double, libm expf/logf/sqrtf. */
#define T float
#define S f
#define ACC double
#define EXP expf
#define LOG logf
#define SQRT sqrtf
#define FABS fabsf
#define TMIN FLT_MIN
#define TEPS FLT_EPSILON
#include "sla2_oracle_body.h"
#undef T
#undef S
#undef ACC
#undef EXP
#undef LOG
#undef SQRT
#undef FABS
#undef TMIN
#undef TEPS

/* double instantiation (Matrix<double>): accumulator long double. */
#define T double
#define S d
#define ACC long double
#define EXP exp
#define LOG log
#define SQRT sqrt
#define FABS fabs
#define TMIN DBL_MIN
#define TEPS DBL_EPSILON
#include "sla2_oracle_body.h"
