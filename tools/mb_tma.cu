// mb_tma.cu -- per-SM TMA load throughput and latency (analysis only, not product).
// 148 CTAs (one per SM); thread 0 of each streams 8 KB boxes (64 cols x 64 rows bf16, SW128, 3-D
// map [heads][rows][128] like the sparse kernel's K / V maps) of randomly chosen key blocks from
// one head (L2-resident working set) into a ring of `depth` 8 KB slots, waiting per slot.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_12675_b200/csrc mb_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace sla2dev;

__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, int depth, int iters,
                                                     int nblk, int heads, unsigned long long* out, int nw, int boxrows) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t fullall[4][32];
    if (threadIdx.x == 0) {
        for (int w = 0; w < 4; ++w)
            for (int s = 0; s < depth; ++s) mbar_init(&fullall[w][s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    // nw > 0: issuer i = lane 0 of warp i; nw < 0: issuer i = lane 8i of warp 0
    const int w = nw > 0 ? (int)(threadIdx.x >> 5) : (int)((threadIdx.x & 31) >> 3);
    const bool is_issuer = nw > 0 ? ((threadIdx.x & 31) == 0 && w < nw) : (threadIdx.x < 32 && (threadIdx.x & 7) == 0 && w < -nw);
    if (nw < 0) nw = -nw;
    const uint32_t boxbytes = 128u * boxrows;
    if (is_issuer) {
        uint64_t* full = fullall[w];
        smem += w * depth * boxbytes;
        uint32_t h = 2654435761u * (blockIdx.x + 1) + 977u * w;
        const int head = blockIdx.x % heads;
        unsigned long long lat_sum = 0;
        const unsigned long long t0 = clock64();
        unsigned long long issued[32];
        for (int it = 0; it < iters + depth; ++it) {
            const int s = it % depth;
            if (it >= depth) {  // retire the load issued depth iterations ago
                mbar_wait(&full[s], (uint32_t)(((it / depth) - 1) & 1));
                lat_sum += clock64() - issued[s];
            }
            if (it < iters) {
                h = h * 1664525u + 1013904223u;
                const int blk = (int)((h >> 8) % (uint32_t)nblk);
                issued[s] = clock64();
                mbar_arrive_expect_tx(&full[s], boxbytes);
                tma_load_3d(smem + s * boxbytes, &tm, (int)((h >> 4) & 1) * 64, blk * 64, head, &full[s]);
            }
        }
        const unsigned long long t1 = clock64();
        if (w == 0) {
            out[blockIdx.x * 2] = t1 - t0;
            out[blockIdx.x * 2 + 1] = lat_sum / iters;
        }
    }
    __syncthreads();
}

int main() {
    const int heads = 12, N = 32768, d = 128;
    void* buf;
    const size_t bytes = (size_t)heads * N * d * 2;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)heads};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)N * d * 2};
    cuuint32_t box[3] = {64, 64, 1}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
    }
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * 2 * sizeof(unsigned long long));
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    std::vector<unsigned long long> h(296);
    CUtensorMap tm128;
    cuuint32_t box128[3] = {64, 128, 1};
    cuTensorMapEncodeTiled(&tm128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box128, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int boxrows : {64, 128}) {
        for (int nw : {1, 4, -4, 8}) {
            for (int depth : {2, 4}) {
                const int anw = nw < 0 ? -nw : nw;
                if (anw * depth * 128 * boxrows > 200 * 1024 || anw > 4 && nw > 0 && false) continue;
                const int iters = 3000;
                const CUtensorMap& m = boxrows == 64 ? tm : tm128;
                const int launch_nw = nw == 8 ? -4 : nw;  // 8 = lanes 0,8,16,24 of warp 0 (same as -4)
                if (nw == 8) continue;
                for (int rep = 0; rep < 2; ++rep)
                    tma_kernel<<<148, 128, 210 * 1024>>>(m, depth, iters, N / 64 - 1, 12, d_out, launch_nw, boxrows);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost);
                double cyc = 0, lat = 0;
                for (int b = 0; b < 148; ++b) {
                    cyc += h[2 * b];
                    lat += h[2 * b + 1];
                }
                cyc /= 148;
                lat /= 148;
                printf("box %3d rows, %d issuers (%s) x depth %d: %.1f B/clk/SM (chip %.0f B/clk), latency %.0f cycles (%s)\n",
                       boxrows, anw, nw < 0 ? "lanes of one warp" : "one lane per warp", depth,
                       (double)anw * iters * 128 * boxrows / cyc, 148.0 * anw * iters * 128 * boxrows / cyc, lat,
                       cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
