// lat_bench.cu -- analysis-only: dependent-chain latency (cycles per op) of the adds the exact
// column mean can use: FADD (f32 + f32), FHADD.BF16 (f32 + bf16, add.rn.f32.bf16), and the
// LDS -> convert -> FADD step. One warp per CTA, 4096 dependent ops.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

__global__ void lat_kernel(int which, int n, float seed, unsigned long long* cyc, float* out) {
    __shared__ unsigned short sh[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = (unsigned short)(0x3f80 + (i & 7));
    __syncthreads();
    float acc = seed;
    const float x = seed * 0.5f;
    const unsigned short h = 0x3f81;
    unsigned long long t0 = clock64();
    if (which == 0) {
#pragma unroll 16
        for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, x);
    } else if (which == 1) {
#pragma unroll 16
        for (int i = 0; i < n; ++i) asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"(h));
    } else if (which == 2) {
#pragma unroll 16
        for (int i = 0; i < n; ++i) {
            unsigned short v = sh[(i * 32 + threadIdx.x) & 4095];
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"(v));
        }
    } else if (which == 3) {  // one 32-bit load (2 columns) -> 2 chains per row
        float acc2 = seed;
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(sh);
#pragma unroll 16
        for (int i = 0; i < n; ++i) {
            const uint32_t w = s32[(i * 32 + threadIdx.x) & 2047];
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"((unsigned short)(w & 0xffff)));
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc2) : "h"((unsigned short)(w >> 16)));
        }
        acc += acc2;
    } else {  // one 64-bit load (4 columns) -> 4 chains per row
        float a1 = seed, a2 = seed, a3 = seed;
        const uint2* s64 = reinterpret_cast<const uint2*>(sh);
#pragma unroll 16
        for (int i = 0; i < n; ++i) {
            const uint2 w = s64[(i * 32 + threadIdx.x) & 1023];
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"((unsigned short)(w.x & 0xffff)));
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(a1) : "h"((unsigned short)(w.x >> 16)));
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(a2) : "h"((unsigned short)(w.y & 0xffff)));
            asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(a3) : "h"((unsigned short)(w.y >> 16)));
        }
        acc += a1 + a2 + a3;
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[threadIdx.x] = acc;
}

extern "C" int lat_bench(int which, int n, unsigned long long* cyc, float* out) {
    lat_kernel<<<1, 32>>>(which, n, 1.0f, cyc, out);
    return (int)cudaDeviceSynchronize();
}
