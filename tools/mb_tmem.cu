// mb_tmem.cu -- microbenchmarks for the sparse-kernel redesign (analysis only, not product):
// per-SM TMEM load bandwidth (tcgen05.ld 32x32b.x32) and MUFU ex2 / F2FP throughput, as a
// function of the number of warps issuing. One CTA per SM, clock64 around the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12675_b200/csrc mb_tmem.cu -o mb_tmem
#include <cstdio>
#include <cuda_runtime.h>

#include "tc.cuh"

using namespace sla2dev;

template <int XN>
__global__ void tmem_ld_kernel(int iters, int nwarps, unsigned long long* out, float* sink) {
    __shared__ uint32_t base_sh;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&base_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = base_sh;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col0 = (uint32_t)((warp >> 2) * 128) & 511;
    float acc = 0.f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (warp < nwarps) {
        for (int it = 0; it < iters; ++it) {
            uint32_t r[4][32];
#pragma unroll
            for (int u = 0; u < XN; ++u) tmem_ld32(tmem + lane_base + col0 + u * 32, r[u]);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; c += 8) acc += __uint_as_float(r[0][c]) + __uint_as_float(r[XN - 1][c]);
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

__global__ void ex2_kernel(int iters, int nwarps, unsigned long long* out, float* sink) {
    const int warp = threadIdx.x >> 5;
    float x[8];
    for (int u = 0; u < 8; ++u) x[u] = -0.001f * (threadIdx.x + u);
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (warp < nwarps) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float y;
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[u]));
                x[u] = y - 1.0f;
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    float s = 0;
    for (int u = 0; u < 8; ++u) s += x[u];
    if (s == 12345.f) sink[threadIdx.x] = s;
}

// F2FP (two fp32 -> packed bf16x2) throughput
__global__ void f2fp_kernel(int iters, int nwarps, unsigned long long* out, float* sink) {
    const int warp = threadIdx.x >> 5;
    float x[8];
    uint32_t acc = 0;
    for (int u = 0; u < 8; ++u) x[u] = 0.001f * (threadIdx.x + u);
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (warp < nwarps) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                uint32_t p = pack_bf16(x[u], x[u + 1]);
                acc ^= p;
                x[u] = __uint_as_float(p & 0xffff0000u);
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345u) sink[threadIdx.x] = (float)acc;
}

int main() {
    unsigned long long* d_out;
    float* sink;
    cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
    cudaMalloc(&sink, 1024 * sizeof(float));
    unsigned long long h[148];
    const int iters = 2000;
    for (int nw : {4, 8, 16}) {
        for (int xn : {1, 2, 4}) {
            if (xn == 1) tmem_ld_kernel<1><<<148, 512>>>(iters, nw, d_out, sink);
            if (xn == 2) tmem_ld_kernel<2><<<148, 512>>>(iters, nw, d_out, sink);
            if (xn == 4) tmem_ld_kernel<4><<<148, 512>>>(iters, nw, d_out, sink);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("err %s\n", cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
            const double bytes = (double)iters * nw * xn * 32 * 32 * 4;
            printf("tmem ld: warps %2d  loads/wait %d  cycles %llu  bytes/clk/SM %.1f\n", nw, xn, h[0],
                   bytes / (double)h[0]);
        }
    }
    for (int nw : {4, 8, 16}) {
        ex2_kernel<<<148, 512>>>(iters, nw, d_out, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        const double ops = (double)iters * nw * 32 * 8;
        printf("ex2: warps %2d  cycles %llu  ex2/clk/SM %.2f\n", nw, h[0], ops / (double)h[0]);
    }
    for (int nw : {4, 8, 16}) {
        f2fp_kernel<<<148, 512>>>(iters, nw, d_out, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        const double ops = (double)iters * nw * 32 * 4;
        printf("f2fp: warps %2d  cycles %llu  pack/clk/SM %.2f\n", nw, h[0], ops / (double)h[0]);
    }
    return 0;
}
