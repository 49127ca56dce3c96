// Exhaustive check of sla2dev::expf_glibc (host build of the device port) against libm expf.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "expf_glibc.cuh"

int main() {
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<unsigned long long> bad(nt, 0);
    std::vector<std::thread> th;
    const uint64_t total = 1ull << 32;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([&, t] {
            const uint64_t lo = total * t / nt, hi = total * (t + 1) / nt;
            for (uint64_t b = lo; b < hi; ++b) {
                const uint32_t u = (uint32_t)b;
                float x;
                std::memcpy(&x, &u, 4);
                const float e = expf(x), m = sla2dev::expf_glibc(x);
                if (std::memcmp(&e, &m, 4) != 0 && !(e != e && m != m)) ++bad[t];
            }
        });
    }
    unsigned long long s = 0;
    for (unsigned t = 0; t < nt; ++t) {
        th[t].join();
        s += bad[t];
    }
    std::printf("expf_glibc vs libm expf over 2^32 inputs: mismatches %llu\n", s);
    return s == 0 ? 0 : 1;
}
