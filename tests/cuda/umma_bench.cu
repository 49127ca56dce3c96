// umma_bench.cu -- analysis-only microbenchmark of tcgen05.mma issue/execution cost
// (kind::f16, M = 128, cta_group::1), one CTA per SM.
//   variant 0: one lane issues, loop of single MMAs into one accumulator
//   variant 1: one lane issues, unrolled x8, one accumulator
//   variant 2: whole warp converged, elect.sync inside the asm, unrolled x8, one accumulator
//   variant 3: like 2 but alternating two independent accumulators
//   variant 4: like 2 but four independent accumulators (N <= 64)
//   variant 5: like 1 but every MMA reads fresh operand addresses (K16 steps over a 128-deep
//              K range, as in a real tile loop) from non-zero data
//   variant 6: the sparse kernel's per-pair mix (form/N ignored): PV (TS B-MN N128) x8,
//              QK (SS K/K N128) x8, HS (SS MN/MN N128) x8, fresh addresses; cycles per MMA
//   variant 7: like 6 but QK writes the TMEM columns PV reads P from (the S-buffer reuse
//              of the kernel: PV(n) then QK(n+2) into the same buffer)
//   variant 8: like 6 without QK (PV x8, HS x8)
//   variant 9: like 6 plus a tcgen05.commit after each group of 8 (as the kernel commits)
//   variant 10: like 9 plus mbarrier wait (already complete) + tcgen05.fence::after_thread_sync
//               before each group (as the kernel waits on P / K / V before issuing)
//   flags (added to the variant): 16 = warps 2-3 load 128 TMEM columns and store 64 in a loop
//   (the softmax's TMEM traffic); 32 = warp 1 streams 32 KB bulk copies global -> smem (the
//   TMA producers' traffic)
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

constexpr int SMEM_B = 160 * 1024;

__global__ void __launch_bounds__(128, 1) umma_bench_kernel(int form, int variant, int n, int reps,
                                                            unsigned long long* cycles, const uint8_t* gbuf) {
    const int flags = variant & ~15;
    variant &= 15;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2, bar3;
    __shared__ volatile int done;
    __shared__ uint32_t tmem_base;
    for (int e = threadIdx.x; e < SMEM_B / 16; e += blockDim.x) {
        const uint32_t h = (uint32_t)e * 2654435761u;
        // bf16 values in [-2, 2): random mantissas, small exponents
        const uint32_t w = ((h & 0x807f807fu) | 0x3f003f00u) ^ ((h >> 7) & 0x00400040u);
        reinterpret_cast<uint4*>(smem)[e] = make_uint4(w, w * 3u, w ^ 0x1234u, w + 0x10001u);
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        mbar_init(&bar3, 1);
        done = 0;
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
        } else if (variant == 5) {
            if (threadIdx.x == 0)
                for (int r = 0; r < reps; r += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t oa = a_mn ? u * 2048 : (u >> 2) * 16384 + (u & 3) * 32;
                        const uint32_t ob = b_mn ? u * 2048 : (u >> 2) * 32768 + (u & 3) * 32;
                        const uint64_t adu = a_mn ? sdesc_sw128(a + oa, 8192, 1024) : sdesc_sw128(a + oa, 16, 1024);
                        const uint64_t bdu = b_mn ? sdesc_sw128(b + ob, 8192, 1024) : sdesc_sw128(b + ob, 16, 1024);
                        if (ts) umma_bf16_ts(d0, t + u * 8, bdu, idesc, 1);
                        else umma_bf16_ss(d0, adu, bdu, idesc, 1);
                    }
                }
        } else if (variant >= 6) {
            const uint32_t id_qk = idesc_bf16(128, 128, false, false), id_pv = idesc_bf16(128, 128, false, true),
                           id_hs = idesc_bf16(128, 128, true, true);
            const uint32_t q = smem_u32(smem), kp = smem_u32(smem + 32768), vv = smem_u32(smem + 98304),
                           ph = smem_u32(smem + 131072);
            const uint32_t dqk = variant == 7 ? t : t + 128;
            const bool cm = variant >= 9, fw = variant >= 10;
            auto group_edge = [&]() {
                if (cm) umma_commit(&bar3);
                if (fw) {
                    mbar_try_wait(&bar, 0);  // bar is never completed here: returns false at once
                    tc_fence_after();
                }
            };
            if (threadIdx.x == 0)
                for (int r = 0; r < reps; r += 24) {
                    group_edge();
#pragma unroll
                    for (int u = 0; u < 8; ++u)  // PV: P from TMEM cols 0.., V MN-major
                        umma_bf16_ts(t + 256, t + (u >> 2) * 64 + (u & 3) * 8,
                                     sdesc_sw128(vv + (u & 3) * 2048 + (u >> 2) * 16384, 8192, 1024), id_pv, 1);
                    group_edge();
                    if (variant != 8) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) {  // QK pair: Q K-major, K pair K-major
                            const uint32_t off = (u >> 2) * 16384 + (u & 3) * 32;
                            umma_bf16_ss(dqk, sdesc_sw128(q + off, 16, 1024), sdesc_sw128(kp + off, 16, 1024), id_qk, 1);
                        }
                    }
                    group_edge();
#pragma unroll
                    for (int u = 0; u < 8; ++u)  // HS: phi(K)^T and V, both MN-major
                        umma_bf16_ss(t + 384, sdesc_sw128(ph + (u & 3) * 2048 + (u >> 2) * 16384, 8192, 1024),
                                     sdesc_sw128(vv + (u & 3) * 2048 + (u >> 2) * 16384, 8192, 1024), id_hs, 1);
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
            done = 1;
        }
    } else if ((flags & 16) && threadIdx.x >= 64) {
        const uint32_t lb = t + ((uint32_t)((threadIdx.x >> 5) & 3) * 32 << 16);
        while (!done) {
            uint32_t r0[32], r1[32], r2[32], r3[32];
            tmem_ld32(lb, r0);
            tmem_ld32(lb + 32, r1);
            tmem_ld32(lb + 64, r2);
            tmem_ld32(lb + 96, r3);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r0[e] ^= r1[e] ^ r2[e] ^ r3[e];
            tmem_st32(lb + 160, r0);
            tmem_st32(lb + 192, r0);
            tmem_st_wait();
        }
    }
    if ((flags & 32) && threadIdx.x == 32) {
        uint32_t ph = 0;
        for (uint64_t it = 0; !done; ++it, ph ^= 1) {
            const uint8_t* src = gbuf + ((it * 32768) & ((64ull << 20) - 1));
            mbar_arrive_expect_tx(&bar2, 32768);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(
                    smem_u32(smem + 98304)),
                "l"(src), "r"(smem_u32(&bar2))
                : "memory");
            mbar_wait(&bar2, ph);
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_free(t, 512);
}

extern "C" int umma_bench(int form, int variant, int n, int reps, int ctas, unsigned long long* cycles,
                          const void* gbuf) {
    cudaFuncSetAttribute(umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_B + 1024);
    umma_bench_kernel<<<ctas, 128, SMEM_B + 1024>>>(form, variant, n, reps, cycles, (const uint8_t*)gbuf);
    return (int)cudaDeviceSynchronize();
}
