// umma_bench.cu -- analysis-only microbenchmark of tcgen05.mma issue/execution cost
// (kind::f16, M = 128, cta_group::1), one CTA per SM.
//   variant 0: one lane issues, loop of single MMAs into one accumulator
//   variant 1: one lane issues, unrolled x8, one accumulator
//   variant 2: whole warp converged, elect.sync inside the asm, unrolled x8, one accumulator
//   variant 3: like 2 but alternating two independent accumulators
//   variant 4: like 2 but four independent accumulators (N <= 64)
// form: 0 SS K/K, 1 SS K/MN, 2 SS MN/MN, 3 TS B-K, 4 TS B-MN
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_2602_12675_b200/csrc/tc.cuh"

using namespace sla2dev;

__device__ __forceinline__ void mma_elect(bool ts, uint32_t d, uint32_t a_tmem, uint64_t ad, uint64_t bd,
                                          uint32_t idesc) {
    if (ts) {
        asm volatile(
            "{\n\t.reg .pred P, q;\n\t"
            "elect.sync _|P, 0xffffffff;\n\t"
            "setp.ne.b32 q, 1, 0;\n\t"
            "@P tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d),
            "r"(a_tmem), "l"(bd), "r"(idesc)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred P, q;\n\t"
            "elect.sync _|P, 0xffffffff;\n\t"
            "setp.ne.b32 q, 1, 0;\n\t"
            "@P tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc)
            : "memory");
    }
}

__global__ void __launch_bounds__(128, 1) umma_bench_kernel(int form, int variant, int n, int reps,
                                                            unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    for (int e = threadIdx.x; e < 65536 / 16; e += blockDim.x) reinterpret_cast<uint4*>(smem)[e] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tmem_base;
    const bool a_mn = form == 2, b_mn = (form == 1 || form == 2 || form == 4), ts = form >= 3;
    const uint32_t idesc = idesc_bf16(128, n, a_mn, b_mn);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint64_t ad = a_mn ? sdesc_sw128(a, 8192, 1024) : sdesc_sw128(a, 16, 1024);
    const uint64_t bd = b_mn ? sdesc_sw128(b, 8192, 1024) : sdesc_sw128(b, 16, 1024);
    const uint32_t d0 = t + 256, d1 = t + 256 + 128, d2 = t + 256 + 64, d3 = t + 256 + 192;
    unsigned long long t0 = 0;
    if (threadIdx.x < 32) {
        t0 = clock64();
        if (variant == 0) {
            if (threadIdx.x == 0)
                for (int r = 0; r < reps; ++r) {
                    if (ts) umma_bf16_ts(d0, t, bd, idesc, 1);
                    else umma_bf16_ss(d0, ad, bd, idesc, 1);
                }
        } else if (variant == 1) {
            if (threadIdx.x == 0)
                for (int r = 0; r < reps; r += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (ts) umma_bf16_ts(d0, t, bd, idesc, 1);
                        else umma_bf16_ss(d0, ad, bd, idesc, 1);
                    }
                }
        } else {
            for (int r = 0; r < reps; r += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t d = variant == 2 ? d0 : variant == 3 ? ((u & 1) ? d1 : d0)
                                                   : ((u & 3) == 0 ? d0 : (u & 3) == 1 ? d2 : (u & 3) == 2 ? d1 : d3);
                    mma_elect(ts, d, t, ad, bd, idesc);
                }
            }
        }
        __syncwarp();
        if (threadIdx.x == 0) {
            umma_commit(&bar);
            mbar_wait(&bar, 0);
            cycles[blockIdx.x] = clock64() - t0;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_free(t, 512);
}

extern "C" int umma_bench(int form, int variant, int n, int reps, int ctas, unsigned long long* cycles) {
    cudaFuncSetAttribute(umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    umma_bench_kernel<<<ctas, 128, 65536 + 1024>>>(form, variant, n, reps, cycles);
    return (int)cudaDeviceSynchronize();
}
