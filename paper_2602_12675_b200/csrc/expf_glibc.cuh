// expf_glibc.cuh -- bit-exact port of glibc 2.39's expf (sysdeps/ieee754/flt-32/e_expf.c, the
// FMA ifunc variant x86_64 selects on FMA-capable hosts), for host and device.
//
// Why: the router's row softmax (matrix.hpp:138-155, called from router.hpp:101) feeds the
// hard top-k; reproducing the reference's mask bit-for-bit needs the same expf results the
// reference gets from libm. Algorithm (public, ARM optimized-routines): x*N/ln2 = k + r with
// N = 32; exp(x) = 2^(k/N) * 2^(r/N), 2^(k/N) from a 32-entry table, 2^(r/N) by a cubic, all
// in double, rounded once to float. Constants are libm's __exp2f_data (verified against the
// bytes of /lib/x86_64-linux-gnu/libm.so.6), and every double op is an explicit
// correctly-rounded intrinsic so nvcc cannot re-associate or contract differently.
// tests/test_expf.py checks this port against the host libm on all 2^32 inputs.
#pragma once
#include <cstdint>
#include <cstring>
#include <cmath>

namespace sla2dev {

#ifdef __CUDACC__
#define SLA2_HD __host__ __device__ __forceinline__
#else
#define SLA2_HD inline
#endif

// 2^(i/32) bit patterns minus (i << 47); libm's __exp2f_data.tab.
#define SLA2_EXPF_TAB                                                                                 \
    {                                                                                                 \
        0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,   \
            0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, \
            0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull, \
            0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull, \
            0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull, \
            0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull, \
            0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull, \
            0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull    \
    }
#ifdef __CUDACC__
static __constant__ uint64_t c_expf_tab[32] = SLA2_EXPF_TAB;
#endif
static const uint64_t h_expf_tab[32] = SLA2_EXPF_TAB;

SLA2_HD uint64_t expf_tab(uint32_t i) {
#ifdef __CUDA_ARCH__
    return c_expf_tab[i];
#else
    return h_expf_tab[i];
#endif
}

SLA2_HD double u64_as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double d;
    std::memcpy(&d, &u, 8);
    return d;
#endif
}
SLA2_HD uint64_t f64_as_u64(double d) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
#endif
}

SLA2_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    volatile double r = a * b;
    return r;
#endif
}
SLA2_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    volatile double r = a + b;
    return r;
#endif
}
SLA2_HD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}

// glibc expf, FMA variant. Special cases as e_expf.c: NaN -> NaN, x > 0x1.62e42ep6 -> +inf,
// x < -0x1.9fe368p6 (incl. -inf) -> +0.
SLA2_HD float expf_glibc(float x) {
    if (x != x) return x + x;
    if (x > 0x1.62e42ep6f) return INFINITY;
    if (x < -0x1.9fe368p6f) return 0.0f;
    const double InvLn2N = 0x1.71547652b82fep+0 * 32;
    const double Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
    const double C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
    const double C2 = 0x1.62e42ff0c52d6p-1 / 32;
    const double xd = static_cast<double>(x);
    const double z = dmul(InvLn2N, xd);
    double kd = dadd(z, Shift);
    const uint64_t ki = f64_as_u64(kd);
    kd = dadd(kd, -Shift);
    const double r = dfma(InvLn2N, xd, -kd);
    uint64_t t = expf_tab(static_cast<uint32_t>(ki % 32));
    t += ki << (52 - 5);
    const double s = u64_as_f64(t);
    const double zz = dfma(C0, r, C1);
    const double r2 = dmul(r, r);
    double y = dfma(C2, r, 1.0);
    y = dfma(zz, r2, y);
    y = dmul(y, s);
#ifdef __CUDA_ARCH__
    return __double2float_rn(y);
#else
    return static_cast<float>(y);
#endif
}

}  // namespace sla2dev
