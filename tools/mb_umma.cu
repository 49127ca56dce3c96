// mb_umma.cu -- completion-throughput microbenchmark of tcgen05.mma shapes the sparse kernel
// uses (analysis only, not product). One CTA per SM, one warp issues `reps` MMAs in groups,
// commits, waits on the mbarrier; clock64 around the whole. Optional concurrent traffic:
// warps 2-3 stream bulk copies L2 -> smem (the TMA producers' smem writes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12675_b200/csrc mb_umma.cu -o bin/mb_umma
#include <cstdio>
#include <cuda_runtime.h>

#include "tc.cuh"

using namespace sla2dev;

constexpr uint32_t SMEM_B = 200 * 1024;

__device__ __forceinline__ void mma_ss(uint32_t kind, uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
    if (kind == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id)
                     : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id)
                 : "memory");
}
__host__ __device__ constexpr uint32_t idesc_f8(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
    return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// mode: 0 SS K/K N128 one acc | 1 TS N128 one acc | 2 SS K/K N256 one acc | 3 SS MN/MN N128 |
//       4 SS K/K N128 two accs alternating | 5 kernel pair mix QK8(SS) PV8(TS) HS8(SS MN) |
//       6 f8f6f4 SS MN/MN N128 K32 | 7 SS K/K N64 one acc | 8 pair mix with HS in f8 (4 instr)
//       9 TS N256 one acc
__global__ void __launch_bounds__(256, 1) umma_kernel(int mode, int reps, int traffic, const uint8_t* gsrc,
                                                      unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, tbar;
    __shared__ uint32_t tmem_base;
    __shared__ volatile int stop;
    for (uint32_t e = threadIdx.x; e < SMEM_B / 16; e += blockDim.x) {
        const uint32_t h = e * 2654435761u;
        const uint32_t w = ((h & 0x807f807fu) | 0x3f003f00u) ^ ((h >> 7) & 0x00400040u);
        reinterpret_cast<uint4*>(smem)[e] = make_uint4(w, w * 3u, w ^ 0x1234u, w + 0x10001u);
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&tbar, 1);
        stop = 0;
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tmem_base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 65536), sc = smem_u32(smem + 131072);
        const unsigned long long t0 = clock64();
        if (threadIdx.x == 0) {
            const uint32_t idKK128 = idesc_bf16(128, 128, false, false), idKK256 = idesc_bf16(128, 256, false, false),
                           idKK64 = idesc_bf16(128, 64, false, false), idMM = idesc_bf16(128, 128, true, true),
                           idTS = idesc_bf16(128, 128, false, true), idTS256 = idesc_bf16(128, 256, false, true),
                           idF8 = idesc_f8(128, 128, true, true);
            for (int r = 0; r < reps; r += 24) {
                if (mode == 0 || mode == 2 || mode == 7) {
                    const uint32_t id = mode == 0 ? idKK128 : mode == 2 ? idKK256 : idKK64;
#pragma unroll
                    for (int u = 0; u < 24; ++u) {
                        const uint32_t off = ((u & 7) >> 2) * 16384 + (u & 3) * 32;
                        mma_ss(0, t, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off * 2, 16, 1024), id);
                    }
                } else if (mode == 1 || mode == 9) {
#pragma unroll
                    for (int u = 0; u < 24; ++u)
                        mma_ts(t + 256, t + (u & 7) * 8, sdesc_sw128(sb + (u & 7) * 2048, 8192, 1024),
                               mode == 1 ? idTS : idTS256);
                } else if (mode == 3) {
#pragma unroll
                    for (int u = 0; u < 24; ++u)
                        mma_ss(0, t, sdesc_sw128(sa + (u & 3) * 2048, 8192, 1024),
                               sdesc_sw128(sb + (u & 3) * 2048, 8192, 1024), idMM);
                } else if (mode == 4) {
#pragma unroll
                    for (int u = 0; u < 24; ++u) {
                        const uint32_t off = ((u & 7) >> 2) * 16384 + (u & 3) * 32;
                        mma_ss(0, t + (u & 1) * 128, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024),
                               idKK128);
                    }
                } else if (mode == 5 || mode == 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t off = (u >> 2) * 16384 + (u & 3) * 32;
                        mma_ss(0, t, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024), idKK128);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        mma_ts(t + 256, t + 128 + u * 8, sdesc_sw128(sc + (u & 3) * 2048 + (u >> 2) * 16384, 8192, 1024),
                               idTS);
                    if (mode == 5) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            mma_ss(0, t + 384, sdesc_sw128(sc + 32768 + (u & 3) * 2048, 8192, 1024),
                                   sdesc_sw128(sc + (u & 3) * 2048, 8192, 1024), idMM);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            mma_ss(1, t + 384, sdesc_sw128(sc + 32768 + u * 4096, 8192, 1024),
                                   sdesc_sw128(sc + u * 4096, 8192, 1024), idF8);
                        r -= 4;  // 20 MMAs per group in this mode
                    }
                } else if (mode == 6) {
#pragma unroll
                    for (int u = 0; u < 24; ++u)
                        mma_ss(1, t, sdesc_sw128(sa + (u & 3) * 4096, 8192, 1024),
                               sdesc_sw128(sb + (u & 3) * 4096, 8192, 1024), idF8);
                }
            }
            umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        const unsigned long long t1 = clock64();
        if (threadIdx.x == 0) {
            out[blockIdx.x] = t1 - t0;
            stop = 1;
        }
    } else if (warp == 2 && traffic) {
        // `traffic` bulk copies of 8 KB in flight, global (an L2-resident 1 MB window) -> smem
        // region [160 KB, 160 KB + 8 KB * traffic): the TMA producers' smem writes
        if (threadIdx.x == 64) {
            __shared__ uint64_t tb[8];
            for (int s = 0; s < traffic; ++s) mbar_init(&tb[s], 1);
            fence_barrier_init();
            uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            long n = 0;
            auto issue = [&](int s) {
                mbar_arrive_expect_tx(&tb[s], 8192);
                const uint8_t* src = gsrc + ((size_t)((blockIdx.x * 8191 + n * 37) & 8191) << 13);  // 64 MB window
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(smem + 163840 + s * 8192)),
                    "l"(src), "r"(8192), "r"(smem_u32(&tb[s]))
                    : "memory");
                ++n;
            };
            for (int s = 0; s < traffic; ++s) issue(s);
            int s = 0;
            while (!stop) {
                mbar_wait(&tb[s], ph[s]);
                ph[s] ^= 1;
                issue(s);
                s = (s + 1) % traffic;
            }
            for (int u = 0; u < traffic; ++u) mbar_wait(&tb[u], ph[u]);
            out[148 + blockIdx.x] = n;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_free(t, 512);
    }
}

int main() {
    unsigned long long* d_out;
    uint8_t* g;
    cudaMalloc(&d_out, 2 * 148 * sizeof(unsigned long long));
    cudaMalloc(&g, 64 << 20);
    cudaMemset(g, 1, 64 << 20);
    cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_B + 1024);
    const char* names[] = {"SS K/K N128 1acc",   "TS N128 1acc",        "SS K/K N256 1acc", "SS MN/MN N128",
                           "SS N128 2acc alt",   "pair mix QK8 PV8 HS8", "f8 SS MN N128 K32", "SS K/K N64 1acc",
                           "pair mix, HS f8 x4", "TS N256 1acc"};
    const double flop_per[] = {2.0 * 128 * 128 * 16, 2.0 * 128 * 128 * 16, 2.0 * 128 * 256 * 16, 2.0 * 128 * 128 * 16,
                               2.0 * 128 * 128 * 16, 2.0 * 128 * 128 * 16, 2.0 * 128 * 128 * 32, 2.0 * 128 * 64 * 16,
                               2.0 * 128 * 128 * 16, 2.0 * 128 * 256 * 16};
    const int reps = 24 * 400;
    for (int traffic : {0, 1, 2, 4, 6}) {
        for (int mode = 0; mode < 10; ++mode) {
            if (traffic && mode != 0 && mode != 1 && mode != 3 && mode != 5) continue;
            umma_kernel<<<148, 256, SMEM_B + 1024>>>(mode, reps, traffic, g, d_out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d err %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            unsigned long long h[296];
            cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
            int nmma = mode == 8 ? reps / 24 * 20 : reps;
            double cyc = (double)h[0] / nmma;
            double fpc = (mode == 8 ? (16 * 2.0 * 128 * 128 * 16 + 4 * 2.0 * 128 * 128 * 32) / 20 : flop_per[mode]) / cyc;
            printf("traffic %d  %-22s cycles/MMA %6.1f  flop/clk %7.0f (peak bf16 8192)%s", traffic, names[mode], cyc,
                   fpc, traffic ? "" : "\n");
            if (traffic) printf("  copies %.1f B/clk\n", (double)h[148] * 8192.0 / (double)h[0]);
        }
    }
    return 0;
}
