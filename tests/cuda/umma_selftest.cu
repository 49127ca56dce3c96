// umma_selftest.cu -- test-only sm_100a kernels that pin the tcgen05 / TMA encodings used by
// the product kernels (descriptor bit layout, SWIZZLE_128B addressing for K-major and
// MN-major operands, bf16 and int8 kinds, TMEM load layout). Built into
// tests/cuda/libumma_selftest.so by tests/cuda/Makefile; exercised by tests/test_gpu_umma.py.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_2602_12675_b200/csrc/expf_glibc.cuh"
#include "../../paper_2602_12675_b200/csrc/tc.cuh"

using namespace sla2dev;

// mode 0: bf16  D[128x64]  = A[128x128](K-major) * B[64x128]^T (K-major)
// mode 1: bf16  D[128x128] = A[128x64](K-major)  * B[64x128]   (B MN-major, stored K x N)
// mode 2: bf16  D[128x128] = A^T where A stored [64 x 128] (MN-major), * B[64x128] (MN-major)
// mode 3: int8  D[128x64]  = A[128x128](K-major) * B[64x128]^T (K-major), s32
// mode 4: int8  D[128x128] = A[128x64](K-major)  * B[64x128]   (B MN-major), s32
// mode 5: bf16  D[128x128] = A[128x128](K-major) * B[128x128] (B MN-major, stored K x N)
__global__ void __launch_bounds__(128, 1) umma_selftest_kernel(int mode, const void* A, const void* B, void* D) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;              // 32 KB
    uint8_t* sB = smem + 32768;      // 32 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;

    int M = 128, N = 64, K = 128;
    bool a_mn = false, b_mn = false, s8 = false;
    switch (mode) {
        case 0: N = 64; K = 128; break;
        case 1: N = 128; K = 64; b_mn = true; break;
        case 2: N = 128; K = 64; a_mn = true; b_mn = true; break;
        case 3: N = 64; K = 128; s8 = true; break;
        case 4: N = 128; K = 64; b_mn = true; s8 = true; break;
        case 5: N = 128; K = 128; b_mn = true; break;
    }
    const int esz = s8 ? 1 : 2;
    const int atom_elems = 128 / esz;  // elements per 128-B swizzle row

    // ---- fill A
    if (!a_mn) {  // A stored [M][K] row-major, K-major SW128 atoms of [M rows][atom_elems]
        for (int i = tid; i < M * K; i += blockDim.x) {
            int r = i / K, c = i % K;
            int atom = c / atom_elems, cc = c % atom_elems;
            uint32_t off = atom * (M * 128) + (s8 ? sw128_off_b(r, cc) : sw128_off(r, cc));
            if (s8) sA[off] = reinterpret_cast<const uint8_t*>(A)[i];
            else *reinterpret_cast<uint16_t*>(sA + off) = reinterpret_cast<const uint16_t*>(A)[i];
        }
    } else {  // A stored [K][M] row-major (MN contiguous), MN-major atoms of [K rows][atom_elems]
        for (int i = tid; i < K * M; i += blockDim.x) {
            int kr = i / M, m = i % M;
            int atom = m / atom_elems, mm = m % atom_elems;
            uint32_t off = atom * (K * 128) + (s8 ? sw128_off_b(kr, mm) : sw128_off(kr, mm));
            if (s8) sA[off] = reinterpret_cast<const uint8_t*>(A)[i];
            else *reinterpret_cast<uint16_t*>(sA + off) = reinterpret_cast<const uint16_t*>(A)[i];
        }
    }
    // ---- fill B
    if (!b_mn) {  // B stored [N][K]
        for (int i = tid; i < N * K; i += blockDim.x) {
            int r = i / K, c = i % K;
            int atom = c / atom_elems, cc = c % atom_elems;
            uint32_t off = atom * (N * 128) + (s8 ? sw128_off_b(r, cc) : sw128_off(r, cc));
            if (s8) sB[off] = reinterpret_cast<const uint8_t*>(B)[i];
            else *reinterpret_cast<uint16_t*>(sB + off) = reinterpret_cast<const uint16_t*>(B)[i];
        }
    } else {  // B stored [K][N]
        for (int i = tid; i < K * N; i += blockDim.x) {
            int kr = i / N, n = i % N;
            int atom = n / atom_elems, nn = n % atom_elems;
            uint32_t off = atom * (K * 128) + (s8 ? sw128_off_b(kr, nn) : sw128_off(kr, nn));
            if (s8) sB[off] = reinterpret_cast<const uint8_t*>(B)[i];
            else *reinterpret_cast<uint16_t*>(sB + off) = reinterpret_cast<const uint16_t*>(B)[i];
        }
    }
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp_id() == 0) tmem_alloc(&tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;

    if (tid == 0) {
        const int UK = s8 ? 32 : 16;  // K per instruction
        const uint32_t idesc = s8 ? idesc_s8(M, N, a_mn, b_mn) : idesc_bf16(M, N, a_mn, b_mn);
        for (int s = 0; s < K / UK; ++s) {
            const int kk = s * UK;  // element offset along K
            uint64_t ad, bd;
            if (!a_mn) ad = sdesc_sw128(smem_u32(sA) + (kk / atom_elems) * (M * 128) + (kk % atom_elems) * esz, 16, 1024);
            else ad = sdesc_sw128(smem_u32(sA) + kk * 128, K * 128, 1024);
            if (!b_mn) bd = sdesc_sw128(smem_u32(sB) + (kk / atom_elems) * (N * 128) + (kk % atom_elems) * esz, 16, 1024);
            else bd = sdesc_sw128(smem_u32(sB) + kk * 128, K * 128, 1024);
            if (s8) umma_s8_ss(tbase, ad, bd, idesc, s > 0);
            else umma_bf16_ss(tbase, ad, bd, idesc, s > 0);
        }
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    // each warp reads its 32 lanes (rows), N columns
    const int row = warp_id() * 32 + lane_id();
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + ((warp_id() * 32) << 16) + c0, r);
        tmem_ld_wait();
        for (int c = 0; c < 32; ++c) reinterpret_cast<uint32_t*>(D)[row * N + c0 + c] = r[c];
    }
    tc_fence_before();
    __syncthreads();
    if (warp_id() == 0) tmem_free(tbase, 256);
}

// TMA check: load one [64 rows x 64 cols] bf16 box with SWIZZLE_128B from a [rows x cols]
// row-major tensor at (x, y) and dump the raw 8 KB of shared memory.
__global__ void tma_selftest_kernel(const __grid_constant__ CUtensorMap map, int x, int y, uint8_t* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, 8192);
        tma_load_2d(smem, &map, x, y, &bar);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) out[i] = smem[i];
}

// TS check: A [128 x K] bf16 written into TMEM by the threads (lane = row, 2 elements per
// 32-bit column, element k in the low half of column k/2 when k is even), B from smem.
//   mode 0: K = 128, B = [64 x 128] K-major   -> D [128 x 64]  = A * B^T   (the QK shape)
//   mode 1: K = 64,  B = [64 x 128] MN-major  -> D [128 x 128] = A * B     (the PV shape)
__global__ void __launch_bounds__(128, 1) umma_ts_selftest_kernel(int mode, const uint16_t* A, const uint16_t* B,
                                                                  float* D) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sB = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    const int K = mode == 0 ? 128 : 64, N = mode == 0 ? 64 : 128;
    if (mode == 0) {
        for (int i = tid; i < N * K; i += 128) {
            int r = i / K, c = i % K;
            *reinterpret_cast<uint16_t*>(sB + (c / 64) * (N * 128) + sw128_off(r, c % 64)) = B[i];
        }
    } else {
        for (int i = tid; i < K * N; i += 128) {
            int kr = i / N, n = i % N;
            *reinterpret_cast<uint16_t*>(sB + (n / 64) * (K * 128) + sw128_off(kr, n % 64)) = B[i];
        }
    }
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp_id() == 0) tmem_alloc(&tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    const uint32_t lane_base = (warp_id() * 32) << 16;
    // A row `tid` -> TMEM columns [128, 128 + K/2)
    for (int c0 = 0; c0 < K / 2; c0 += 32) {
        uint32_t w[32];
        for (int c = 0; c < 32; ++c)
            w[c] = (uint32_t)A[tid * K + 2 * (c0 + c)] | ((uint32_t)A[tid * K + 2 * (c0 + c) + 1] << 16);
        tmem_st32(tbase + lane_base + 128 + c0, w);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint32_t idesc = idesc_bf16(128, N, false, mode == 1);
        for (int s = 0; s < K / 16; ++s) {
            uint64_t bd = mode == 0 ? sdesc_sw128(smem_u32(sB) + (s / 4) * (N * 128) + (s % 4) * 32, 16, 1024)
                                    : sdesc_sw128(smem_u32(sB) + s * 16 * 128, K * 128, 1024);
            umma_bf16_ts(tbase, tbase + 128 + s * 8, bd, idesc, s > 0);
        }
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    __syncwarp();
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + lane_base + c0, r);
        tmem_ld_wait();
        for (int c = 0; c < 32; ++c) D[tid * N + c0 + c] = __uint_as_float(r[c]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp_id() == 0) tmem_free(tbase, 256);
}
extern "C" int umma_ts_selftest(int mode, const void* A, const void* B, void* D) {
    cudaFuncSetAttribute(umma_ts_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024);
    umma_ts_selftest_kernel<<<1, 128, 33 * 1024>>>(mode, (const uint16_t*)A, (const uint16_t*)B, (float*)D);
    return (int)cudaDeviceSynchronize();
}

// Device expf_glibc over a host-chosen range of float bit patterns [lo, lo + n).
__global__ void expf_selftest_kernel(uint32_t lo, uint32_t n, float* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = expf_glibc(__uint_as_float(lo + i));
}
extern "C" int expf_selftest(uint32_t lo, uint32_t n, float* out) {
    expf_selftest_kernel<<<1184, 256>>>(lo, n, out);
    return (int)cudaDeviceSynchronize();
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int umma_selftest(int mode, const void* A, const void* B, void* D) {
    cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
    umma_selftest_kernel<<<1, 128, 66 * 1024 + 1024>>>(mode, A, B, D);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}

extern "C" int tma_selftest(const void* src, long rows, long cols, int x, int y, void* out) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return -1;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((PFN_encodeTiled)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src), dims,
                                       strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -2;
    cudaFuncSetAttribute(tma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 9 * 1024 + 1024);
    tma_selftest_kernel<<<1, 128, 9 * 1024 + 1024>>>(map, x, y, (uint8_t*)out);
    return (int)cudaDeviceSynchronize();
}
