// analysis only: are FFMA2(a, b, -0) and FADD2 bit-identical to scalar mul.rn / add.rn?
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float* a, const float* b, const float* c, uint32_t* bad, int n, unsigned long long nz) {
    int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (i + 1 >= n) return;
    unsigned long long A = *reinterpret_cast<const unsigned long long*>(a + i);
    unsigned long long B = *reinterpret_cast<const unsigned long long*>(b + i);
    unsigned long long Cc = *reinterpret_cast<const unsigned long long*>(c + i);
    unsigned long long P, S;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(P) : "l"(A), "l"(B), "l"(nz));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(S) : "l"(P), "l"(Cc));
    for (int e = 0; e < 2; ++e) {
        float p = __fmul_rn(a[i + e], b[i + e]);
        float s = __fadd_rn(p, c[i + e]);
        uint32_t pg = (uint32_t)(P >> (32 * e)), sg = (uint32_t)(S >> (32 * e));
        if (pg != __float_as_uint(p)) atomicAdd(&bad[0], 1);
        if (sg != __float_as_uint(s)) atomicAdd(&bad[1], 1);
    }
}
int main() {
    const int n = 1 << 24;
    float *a, *b, *c; uint32_t* bad;
    cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&c, n * 4); cudaMallocManaged(&bad, 8);
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
    for (int i = 0; i < n; ++i) {
        a[i] = (float)((int64_t)(rnd() % 2000001) - 1000000) / 123456.0f;
        b[i] = (float)((int64_t)(rnd() % 2000001) - 1000000) / 98765.0f;
        c[i] = (float)((int64_t)(rnd() % 2000001) - 1000000) / 4321.0f;
    }
    bad[0] = bad[1] = 0;
    k<<<n / 2 / 256, 256>>>(a, b, c, bad, n, 0x8000000080000000ull);
    cudaDeviceSynchronize();
    printf("ffma2(-0) vs mul.rn mismatches: %u, fadd2 vs add.rn mismatches: %u of %d\n", bad[0], bad[1], n);
    return 0;
}
