// capi.cu -- the C ABI of libsla2_b200.so (include/sla2_capi.h): host-side validation with
// the reference's error classes, workspace carving, TMA descriptor creation, and the launch
// sequence of the forward pass. No compute happens on the host and there is no CPU fallback.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/sla2_capi.h"
#include "kernels.h"

using namespace sla2dev;

namespace {

thread_local std::string g_last_error;
thread_local int g_launches = 0;

// optional stage timing: events [0] start, [1] after router, [2] after linear prep, [3] end,
// and timeline points on whichever stream reaches them: [4] mu ready, [5] query side done,
// [6] key prep done, [7] router back half done, [8] linear precompute done
constexpr int NEV = 9;
thread_local bool g_timing = false;
thread_local cudaEvent_t g_ev[NEV] = {};
thread_local int g_ev_dev = -1;  // device the timing events belong to
thread_local bool g_ev_recorded = false;
thread_local unsigned g_ev_mask = 0;
// set by sla2_forward around its sla2_router call: the router records it once mu is ready
thread_local cudaEvent_t g_mu_ready = nullptr;
void mark(int i, cudaStream_t st) {
    if (!g_timing) return;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != g_ev_dev) {  // events are per device: recreate them on a device switch
        for (auto& e : g_ev)
            if (e) {
                cudaEventDestroy(e);
                e = nullptr;
            }
        g_ev_dev = dev;
    }
    if (!g_ev[i]) cudaEventCreate(&g_ev[i]);
    cudaEventRecord(g_ev[i], st);
    if (i == 0) g_ev_mask = 0;
    g_ev_mask |= 1u << i;
    if (i == 3) g_ev_recorded = true;
}

sla2_status fail(sla2_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

#define SLA2_CUDA_TRY(expr)                                                                   \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(SLA2_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// ---------------------------------------------------------------- device check
sla2_status check_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return fail(SLA2_CUDA_ERROR, "no CUDA device (libsla2_b200 has no CPU fallback)");
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(SLA2_CUDA_ERROR, "libsla2_b200 is built for sm_100a (B200); device is sm_" +
                                         std::to_string(major) + std::to_string(minor));
    return SLA2_OK;
}

// ---------------------------------------------------------------- TMA descriptors
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    });
    return fn;
}

struct MapKey {
    const void* ptr;
    uint64_t rows, cols;
    uint32_t box_x, box_y, elem;
    bool swz;
    uint64_t heads;  // 0: 2-D map; else 3-D [heads][rows][cols]
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && box_x == o.box_x && box_y == o.box_y &&
               elem == o.elem && swz == o.swz && heads == o.heads;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        return std::hash<const void*>()(k.ptr) ^ (k.rows * 1315423911u) ^ (k.cols << 7) ^ (k.box_x << 17) ^
               (k.box_y << 23) ^ k.elem ^ (k.heads << 29);
    }
};

// 2-D row-major [rows][cols] tensor of `elem`-byte elements, box (box_x cols, box_y rows),
// SWIZZLE_128B. Cached: descriptors are immutable for a given pointer/shape.
bool make_map(CUtensorMap* out, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_x, uint32_t box_y,
              uint32_t elem, bool swizzle128 = true) {
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    MapKey key{ptr, rows, cols, box_x, box_y, elem, swizzle128, 0};
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *out = it->second;
            return true;
        }
    }
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * elem};
    cuuint32_t box[2] = {box_x, box_y};
    cuuint32_t es[2] = {1, 1};
    const CUtensorMapDataType dt = elem == 2   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                   : elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    CUresult r = fn(out, dt, 2, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *out);
    return true;
}

// 3-D [heads][rows][cols] tensor (rows = N per head), box (box_x cols, box_y rows, 1 head):
// a box never crosses a head, so a ragged N (N % box_y != 0) reads zeros past the head's last
// row and a store drops them.
bool make_map3(CUtensorMap* out, const void* ptr, uint64_t heads, uint64_t rows, uint64_t cols, uint32_t box_x,
               uint32_t box_y, uint32_t elem, bool swizzle128 = true) {
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    MapKey key{ptr, rows, cols, box_x, box_y, elem, swizzle128, heads};
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *out = it->second;
            return true;
        }
    }
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {cols, rows, heads};
    cuuint64_t strides[2] = {cols * elem, rows * cols * elem};
    cuuint32_t box[3] = {box_x, box_y, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapDataType dt = elem == 2   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                   : elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    CUresult r = fn(out, dt, 3, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *out);
    return true;
}

// ---------------------------------------------------------------- geometry + workspace
struct Geo {
    int64_t B, H, BH, N, d, bq, bk, tm, tn, kappa;
    bool bf16, quant;
    bool fp8;  // SLA2_QUANT_FP8PV: E4M3 P / V / phi(K~) in the sparse kernel (tolerance mode)
    int nchunk;
};

Geo geometry(const sla2_fwd_params* p) {
    Geo g{};
    g.B = p->B;
    g.H = p->H;
    g.BH = p->B * p->H;
    g.N = p->N;
    g.d = p->d;
    g.bq = p->bq;
    g.bk = p->bk;
    // ceil: a ragged N (bf16 path) has a partial last query / key block
    g.tm = p->bq ? (p->N + p->bq - 1) / p->bq : 0;
    g.tn = p->bk ? (p->N + p->bk - 1) / p->bk : 0;
    g.kappa = sla2_topk_budget(p->k_percent, g.tn);
    g.bf16 = p->dtype == SLA2_BF16;
    g.quant = p->quant == SLA2_QUANT_INT8;
    g.fp8 = p->quant == SLA2_QUANT_FP8PV && g.bf16;
    if (g.bf16) {
        // Htot partial chunks of 22 key blocks (kphi_htot_kernel, 2 CTAs per SM): at cfg2, 12 heads
        // x 24 chunks = 288 CTAs, one wave on 148 SMs. Depends on tn only, so a head's Htot (and
        // the output) is bit-identical however many heads share a call. (Measured at cfg2:
        // 8 -> 0.654-0.662 ms, 12 -> 0.641-0.644, 22 -> 0.637-0.649, 32 / 43 slower.)
        constexpr int64_t per = 22;  // (re-measured after the router changes: 12 / 16 / 32 not faster)
        g.nchunk = (int)((g.tn + per - 1) / per);
    } else {
        g.nchunk = (int)std::max<int64_t>(1, std::min<int64_t>(64, (g.N + 511) / 512));
    }
    return g;
}

struct Carver {
    uint8_t* base;
    size_t off = 0;
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

struct Workspace {
    float* mu;
    double* mu_part;
    float* qp;
    float* kp;
    float* qbar;
    float* kbar;
    int32_t* idx;
    void* phik;
    float* zblk;
    float* ztot;
    float* hpart;
    float* htot;
    void* htot16;
    void* phiq;  // bf16 path: phi(Q) rows, TMA-loaded by the sparse kernel
    void* ol;    // bf16 path: the linear branch's O_l rows (sparse_fa.cu), [BH][N][d]
    int8_t *qc, *kc, *vct;
    float *qs, *ks, *vs;
    uint8_t *v8, *phi8;  // FP8 P/V mode: E4M3 V and phi(K~) [BH][N][d]
    uint32_t* vamax;     // FP8 P/V mode: [BH] max |V|
    int32_t* cnt;
    int* flag;
};

size_t carve(const Geo& g, void* base, Workspace* w) {
    Carver c{reinterpret_cast<uint8_t*>(base)};
    Workspace t{};
    t.mu = c.take<float>(g.BH * g.d);
    t.mu_part = c.take<double>(g.BH * ((g.N + 255) / 256) * g.d);
    t.qp = c.take<float>(g.BH * g.tm * g.d);
    t.kp = c.take<float>(g.BH * ((g.tn + 3) & ~int64_t(3)) * g.d);  // transposed rows padded to 4 keys
    t.qbar = c.take<float>(g.BH * g.tm * g.d);
    t.kbar = c.take<float>(g.BH * g.tn * g.d);
    t.idx = c.take<int32_t>(g.BH * g.tm * std::max<int64_t>(g.kappa, g.tn));
    t.cnt = c.take<int32_t>(g.BH * g.tm);
    t.flag = c.take<int>(4);
    t.phik = c.take<uint8_t>(g.BH * g.N * g.d * (g.bf16 ? 2 : 4));
    t.zblk = c.take<float>(g.BH * g.tn * g.d);
    t.ztot = c.take<float>(g.BH * g.d);
    t.hpart = c.take<float>(g.BH * g.nchunk * g.d * g.d);
    t.htot = c.take<float>(g.BH * g.d * g.d);
    t.htot16 = c.take<uint16_t>(g.BH * g.d * g.d);
    t.phiq = g.bf16 ? c.take<uint16_t>(g.BH * g.N * g.d) : nullptr;
    t.ol = (g.bf16 && g.quant) ? c.take<uint16_t>(g.BH * g.N * g.d) : nullptr;  // QAT: linear-branch O_l
    if (g.fp8) {
        t.v8 = c.take<uint8_t>(g.BH * g.N * g.d);
        t.phi8 = c.take<uint8_t>(g.BH * g.N * g.d);
        t.vamax = c.take<uint32_t>(g.BH);
    }
    if (g.quant) {
        t.qc = c.take<int8_t>(g.BH * g.N * g.d);
        t.kc = c.take<int8_t>(g.BH * g.N * g.d);
        t.vct = c.take<int8_t>(g.BH * g.N * g.d);
        t.qs = c.take<float>(g.BH * g.tm);
        t.ks = c.take<float>(g.BH * g.tn);
        t.vs = c.take<float>(g.BH * g.tn);
    }
    if (w) *w = t;
    return c.off + 256;
}

// TMA view of K for the serial column-mean kernels, boxes of 128 rows x one 128-byte segment:
// bf16 3-D [BH][N][d] (colmean_tr_kernel, any N: rows past N read as zeros, which leave the
// serial sum unchanged), fp32 2-D [B*H*N][d] (colmean_tma_kernel, N % 128 == 0).
const CUtensorMap* colmean_map(CUtensorMap* m, const void* k, bool bf16, int64_t BH, int64_t N, int64_t d) {
    const uint32_t cols = bf16 ? 64 : 32;
    if (d % cols != 0) return nullptr;
    if (bf16) return make_map3(m, k, (uint64_t)BH, (uint64_t)N, (uint64_t)d, cols, 128, 2, false) ? m : nullptr;
    if (N % 128 != 0) return nullptr;
    return make_map(m, k, (uint64_t)(BH * N), (uint64_t)d, cols, 128, 4, false) ? m : nullptr;
}

float inv_sqrt(int64_t d) {
    // T(1) / std::sqrt(static_cast<T>(d)) for T = float (router.hpp:100, attention.hpp:377)
    volatile float fd = (float)d;
    volatile float s = std::sqrt((float)fd);
    volatile float r = 1.0f / s;
    return r;
}

}  // namespace

namespace sla2dev {
void timeline_mark(int slot, cudaStream_t st) { mark(slot, st); }

static int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

cudaStream_t aux_stream(int slot, int prio) {
    thread_local std::unordered_map<int64_t, cudaStream_t> streams;
    const int64_t key = ((int64_t)current_device() << 16) | (int64_t)(slot & 0xffff);
    auto it = streams.find(key);
    if (it != streams.end()) return it->second;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s = nullptr;
    cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio > 0 ? hi : prio < 0 ? lo : 0);
    streams.emplace(key, s);
    return s;
}

cudaEvent_t aux_event(int slot) {
    thread_local std::unordered_map<int64_t, cudaEvent_t> events;
    const int64_t key = ((int64_t)current_device() << 16) | (int64_t)(slot & 0xffff);
    auto it = events.find(key);
    if (it != events.end()) return it->second;
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    events.emplace(key, e);
    return e;
}

cudaError_t ensure_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> done[64];  // per device: func -> largest size set
    const int dev = current_device() & 63;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = done[dev].find(func);
        if (it != done[dev].end() && it->second >= bytes) return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    int& m = done[dev][func];
    if (bytes > m) m = bytes;
    return cudaSuccess;
}
}  // namespace sla2dev

// =============================================================================================
extern "C" {

const char* sla2_last_error(void) { return g_last_error.c_str(); }
int32_t sla2_last_launch_count(void) { return g_launches; }
const char* sla2_version(void) { return "sla2_b200 0.1.0 sm_100a"; }

void sla2_enable_stage_timing(int32_t enable) { g_timing = enable != 0; }

int32_t sla2_last_stage_ms(float* out, int32_t n) {
    if (!g_ev_recorded || !out || n <= 0) return 0;
    cudaEventSynchronize(g_ev[3]);
    float ms[4 + NEV - 4] = {};
    cudaEventElapsedTime(&ms[0], g_ev[0], g_ev[1]);
    cudaEventElapsedTime(&ms[1], g_ev[1], g_ev[2]);
    cudaEventElapsedTime(&ms[2], g_ev[2], g_ev[3]);
    cudaEventElapsedTime(&ms[3], g_ev[0], g_ev[3]);
    for (int i = 4; i < NEV; ++i) {
        ms[i] = -1.0f;
        if (g_ev_mask & (1u << i)) {
            cudaEventSynchronize(g_ev[i]);
            cudaEventElapsedTime(&ms[i], g_ev[0], g_ev[i]);
        }
    }
    const int m = n < NEV ? n : NEV;
    for (int i = 0; i < m; ++i) out[i] = ms[i];
    return m;
}

void sla2_default_params(sla2_fwd_params* p, int64_t B, int64_t H, int64_t N, int64_t d) {
    std::memset(p, 0, sizeof(*p));
    p->B = B;
    p->H = H;
    p->N = N;
    p->d = d;
    p->bq = 128;
    p->bk = 64;
    p->k_percent = 3.0;
    p->dtype = SLA2_BF16;
    p->quant = SLA2_QUANT_NONE;
    p->smooth = 1;
    p->exact_mu = 1;
    p->tau = 0.1f;
}

int64_t sla2_topk_budget(double k_percent, int64_t tn) {
    // router.hpp:36-40
    const double r = (double)std::llround(k_percent / 100.0 * (double)tn) * 1.0;
    const int64_t kappa = (int64_t)(r > 1.0 ? r : 1.0);
    return kappa < tn ? kappa : tn;
}

// Checks the reference's own prologues make (shapes, budget, tau) plus the dtype/quant enums;
// enough for the router entry points, which have no kernel-geometry limits.
static sla2_status check_common(const sla2_fwd_params* p, bool hard_budget = true) {
    g_last_error.clear();
    if (!p) return fail(SLA2_CONTRACT_ERROR, "params is NULL");
    if (p->B <= 0 || p->H <= 0 || p->N <= 0 || p->d <= 0)
        return fail(SLA2_SHAPE_ERROR, "B, H, N, d must be positive");
    if (p->bq <= 0 || p->bk <= 0) return fail(SLA2_SHAPE_ERROR, "block sizes must be positive");
    if ((p->N % p->bq != 0 || p->N % p->bk != 0) &&
        !(p->dtype == SLA2_BF16 && p->quant != SLA2_QUANT_INT8 && p->d == 128 && p->bq == 128 && p->bk == 64))
        // the reference's rule (attention.hpp:39-41); the ragged extension (partial last blocks,
        // SURVEY.md 8f item 2) exists on the bf16 tcgen05 path only
        return fail(SLA2_SHAPE_ERROR, "AttentionInputs: N must be divisible by bq and bk");
    if (hard_budget && !(p->k_percent > 0.0 && p->k_percent <= 100.0))
        return fail(SLA2_SHAPE_ERROR, "hard_topk: k_percent must be in (0, 100]");  // router.hpp:108-110
    if (!(p->tau > 0.0f)) return fail(SLA2_NUMERIC_ERROR, "RouterParams: tau must be positive");  // router.hpp:32
    if (p->dtype != SLA2_F32 && p->dtype != SLA2_BF16) return fail(SLA2_CONTRACT_ERROR, "unknown dtype");
    if (p->quant != SLA2_QUANT_NONE && p->quant != SLA2_QUANT_INT8 && p->quant != SLA2_QUANT_FP8PV)
        return fail(SLA2_CONTRACT_ERROR, "unknown quant mode");
    if (p->quant == SLA2_QUANT_FP8PV && p->dtype != SLA2_BF16)
        return fail(SLA2_CONTRACT_ERROR, "FP8 P/V mode runs on the bf16 inputs path");
    if (p->N * p->B * p->H > (int64_t)INT32_MAX)
        return fail(SLA2_CONTRACT_ERROR, "B*H*N exceeds the 2^31 row limit of the TMA descriptors");
    return SLA2_OK;
}

sla2_status sla2_check_params(const sla2_fwd_params* p) {
    sla2_status s = check_common(p);
    if (s != SLA2_OK) return s;
    if (p->dtype == SLA2_BF16) {
        if (p->d != 128 || p->bq != 128 || p->bk != 64)
            return fail(SLA2_CONTRACT_ERROR,
                        "bf16 tcgen05 kernels are built for d = 128, bq = 128, bk = 64 (PAPER.md:476)");
    } else {
        if (p->quant != SLA2_QUANT_NONE)
            return fail(SLA2_CONTRACT_ERROR, "INT8 QAT mode runs on the bf16 inputs path");
        if (p->d > 128 || p->bk > 128 || p->bq > 256 || p->bq < 1 || (256 % p->bq) != 0)
            return fail(SLA2_CONTRACT_ERROR, "fp32 path: d <= 128, bk <= 128, bq a power of two <= 256");
        // per-thread register arrays of the CUDA-core kernel: TPR = 256 / bq threads per query
        // row hold ceil(d / TPR) O columns and ceil(bk / TPR) scores, 64 each at most
        const int64_t tpr = p->bq >= 8 ? 256 / p->bq : 32;
        if ((p->d + tpr - 1) / tpr > 64 || (p->bk + tpr - 1) / tpr > 64)
            return fail(SLA2_CONTRACT_ERROR, "fp32 path: ceil(d / (256 / bq)) and ceil(bk / (256 / bq)) must be <= 64");
        if (sparse_f32_smem_bytes((int)p->d, (int)p->bq, (int)p->bk) > 227 * 1024)
            return fail(SLA2_CONTRACT_ERROR, "fp32 path: bq*d + 3*bk*d + bq*bk exceeds shared memory");
    }
    return SLA2_OK;
}

size_t sla2_workspace_size(const sla2_fwd_params* p) {
    if (check_common(p) != SLA2_OK) return 0;  // layout does not depend on kernel limits
    return carve(geometry(p), nullptr, nullptr);
}

// How the linear-branch precompute is scheduled (sla2_forward):
//   dep     fork it onto a second stream off this event (it needs only mu), concurrently with
//           whatever st is still doing; st joins it before the sparse kernel
//   kprep   fork at mu: phi(K~) and z_j (launch_kphi), Htot partials and reduction on the
//           linear stream; the router's pooled keys (launch_kpool) then run on st
//   between run on st right after the fork (the router's back half)
struct LinPlan {
    cudaEvent_t dep = nullptr;
    cudaEvent_t qv_codes = nullptr;  // QAT: Q and V codes were quantized on a side stream (done at this event)
    cudaEvent_t fp8_v = nullptr;     // FP8 P/V: V8 and its per-head scale were made on a side stream
    bool kprep = false;
    bool phiq_ready = false;  // the router front already wrote phi(Q) (bf16 path)
    float* kbar = nullptr;
    std::function<sla2_status(cudaStream_t)> between;
};

// QuantLaunch of the forward's QAT operands (quant_prep_kernel; `which` picks Q / K~ / V).
static QuantLaunch quant_launch(const sla2_fwd_params* p, const Geo& g, const Workspace& w, const void* q,
                                const void* k, const void* v, int which) {
    QuantLaunch qa{};
    qa.B = g.B;
    qa.H = g.H;
    qa.N = (int)g.N;
    qa.d = (int)g.d;
    qa.bq = (int)g.bq;
    qa.bk = (int)g.bk;
    qa.tm = (int)g.tm;
    qa.tn = (int)g.tn;
    qa.q = q;
    qa.k = k;
    qa.v = v;
    qa.mu = w.mu;
    qa.smooth = p->smooth;
    qa.qc = w.qc;
    qa.qs = w.qs;
    qa.kc = w.kc;
    qa.ks = w.ks;
    qa.vct = w.vct;
    qa.vs = w.vs;
    qa.which = which;
    return qa;
}

// Linear-branch precompute then the sparse kernel.
static sla2_status run_linear_and_sparse(const sla2_fwd_params* p, const Geo& g, const Workspace& w, const void* q,
                                         const void* k, const void* v, const float* rho, const int32_t* idx,
                                         const int32_t* cnt, int kstride, void* out, const sla2_fwd_saved* saved,
                                         cudaStream_t st, const LinPlan& plan = LinPlan{}) {
    const float isd = inv_sqrt(g.d);
    CUtensorMap mq, mk, mv, mphi, mht, mpq, mo;
    const uint64_t rows = (uint64_t)(g.BH * g.N);
    if (g.bf16) {
        // per-token tensors as 3-D [BH][N][d] maps (ragged N safe); Htot 2-D
        const uint64_t BH = (uint64_t)g.BH, N = (uint64_t)g.N;
        if (!make_map3(&mq, q, BH, N, g.d, 64, 64, 2) || !make_map3(&mk, k, BH, N, g.d, 64, 64, 2) ||
            !make_map3(&mv, v, BH, N, g.d, 64, 64, 2) || !make_map3(&mphi, w.phik, BH, N, g.d, 64, 64, 2) ||
            !make_map(&mht, w.htot16, (uint64_t)(g.BH * g.d), g.d, 64, 128, 2) ||
            (w.phiq && !make_map3(&mpq, w.phiq, BH, N, g.d, 64, 64, 2)) || !make_map3(&mo, out, BH, N, g.d, 64, 64, 2))
            return fail(SLA2_CUDA_ERROR, "cuTensorMapEncodeTiled failed (pointers must be 16-byte aligned)");
        if (w.phiq && !plan.phiq_ready) SLA2_CUDA_TRY(launch_phiq(q, w.phiq, (int64_t)rows, st, &g_launches));
    }
    LinearLaunch la{};
    la.k = k;
    la.v = v;
    la.bf16 = g.bf16;
    la.BH = g.BH;
    la.N = (int)g.N;
    la.d = (int)g.d;
    la.bk = (int)g.bk;
    la.mu = p->smooth ? w.mu : nullptr;
    la.phik = w.phik;
    la.zblk = w.zblk;
    la.ztot = w.ztot;
    la.hpart = w.hpart;
    la.htot = w.htot;
    la.htot16 = w.htot16;
    la.nchunk = g.nchunk;
    la.tm_phik = &mphi;
    la.tm_v = &mv;
    la.tm_k = (g.bf16 && g.d == 128 && g.bk == 64) ? &mk : nullptr;
    cudaEvent_t dep = plan.dep;
    if (plan.kprep) {
        cudaEvent_t ev_k = aux_event(10);
        // fork at mu: phi(K~), z_j and Htot on the linear stream, beside the router's pooled
        // keys (launch_kpool, below) and back half on st. Forking after the pooled keys instead
        // was measured slower (the router's back half loses more to the concurrent precompute
        // than the pooled keys gain: 0.622 vs 0.619 ms at cfg2)
        la.phik_ready = !(la.tm_k && la.mu);  // the fused kernel computes phi(K~) itself
        SLA2_CUDA_TRY(cudaEventRecord(ev_k, st));
        dep = ev_k;
    }
    cudaEvent_t kc_ready = nullptr;  // QAT: the K~ codes were made on the side stream
    if (dep && g.quant && plan.qv_codes) {
        // the K~ codes need only mu: on the QAT side stream (after its Q / V codes), beside the
        // router's key side, instead of serially between the router and the attention kernels
        cudaStream_t qs = aux_stream(3, -1);
        kc_ready = aux_event(18);
        SLA2_CUDA_TRY(cudaStreamWaitEvent(qs, dep, 0));
        const QuantLaunch qk = quant_launch(p, g, w, q, k, v, 2);
        SLA2_CUDA_TRY(launch_quant_prep(qk, qs, &g_launches));
        SLA2_CUDA_TRY(cudaEventRecord(kc_ready, qs));
    }
    if (dep) {
        // lowest priority (the default level): the router's key side below runs above it
        cudaStream_t lin = aux_stream(1, -1);
        cudaEvent_t lin_done = aux_event(11);
        SLA2_CUDA_TRY(cudaStreamWaitEvent(lin, dep, 0));
        if (plan.kprep && la.phik_ready) SLA2_CUDA_TRY(launch_kphi(la, lin, &g_launches));
        // FP8 P/V: the fused phi(K~) / Htot kernel writes E4M3 phi(K~) directly
        const bool phi8_fused = g.fp8 && la.tm_k && !la.phik_ready;
        if (phi8_fused) la.phi8 = w.phi8;
        SLA2_CUDA_TRY(launch_linear_prep(la, lin, &g_launches));
        if (g.fp8 && (!phi8_fused || !plan.fp8_v))  // the E4M3 operands not made elsewhere
            SLA2_CUDA_TRY(launch_fp8pv_prep(plan.fp8_v ? nullptr : v, phi8_fused ? nullptr : w.phik, w.v8, w.phi8,
                                            w.vamax, g.BH, g.N, lin, &g_launches));
        mark(8, lin);
        SLA2_CUDA_TRY(cudaEventRecord(lin_done, lin));
        // the router's key side on a high-priority stream: the block scheduler serves it ahead of
        // the linear precompute, which otherwise sits at the caller stream's (default) priority
        // (cfg2 forward 0.570 -> 0.557 ms; cfg4 unchanged)
        cudaStream_t rs = aux_stream(5, +1);
        cudaEvent_t ev_f = aux_event(16), ev_j = aux_event(17);
        SLA2_CUDA_TRY(cudaEventRecord(ev_f, st));
        SLA2_CUDA_TRY(cudaStreamWaitEvent(rs, ev_f, 0));
        if (plan.kprep) {
            LinearLaunch lk = la;  // the router's pooled keys: always the exact serial mean
            lk.mu = p->smooth ? w.mu : nullptr;
            SLA2_CUDA_TRY(launch_kpool(lk, plan.kbar, rs, &g_launches));
            mark(6, rs);
        }
        if (plan.between) {
            const sla2_status bs = plan.between(rs);
            if (bs != SLA2_OK) {
                cudaEventRecord(ev_j, rs);
                cudaStreamWaitEvent(st, ev_j, 0);
                cudaStreamWaitEvent(st, lin_done, 0);
                return bs;
            }
            mark(7, rs);
        }
        SLA2_CUDA_TRY(cudaEventRecord(ev_j, rs));
        SLA2_CUDA_TRY(cudaStreamWaitEvent(st, ev_j, 0));
        mark(1, st);  // router done (the linear precompute overlapped it)
        SLA2_CUDA_TRY(cudaStreamWaitEvent(st, lin_done, 0));
    } else {
        SLA2_CUDA_TRY(launch_linear_prep(la, st, &g_launches));
        if (g.fp8) SLA2_CUDA_TRY(launch_fp8pv_prep(v, w.phik, w.v8, w.phi8, w.vamax, g.BH, g.N, st, &g_launches));
    }
    mark(2, st);

    SparseLaunch sa{};
    sa.B = g.B;
    sa.H = g.H;
    sa.N = (int)g.N;
    sa.d = (int)g.d;
    sa.bq = (int)g.bq;
    sa.bk = (int)g.bk;
    sa.tm = (int)g.tm;
    sa.tn = (int)g.tn;
    sa.kv_idx = idx;
    sa.kv_cnt = cnt;
    sa.kstride = kstride;
    sa.kappa = (int)g.kappa;
    sa.rho = rho;
    sa.htot = w.htot;
    sa.htot16 = w.htot16;
    sa.ztot = w.ztot;
    sa.zblk = w.zblk;
    sa.mu = w.mu;
    sa.smooth = p->smooth;
    sa.dense = 0;
    sa.inv_sqrt_d = isd;
    sa.out = out;
    sa.o_s = saved ? saved->o_s : nullptr;
    sa.o_l = saved ? saved->o_l : nullptr;
    sa.big_l = saved ? saved->big_l : nullptr;
    sa.h_blocks = saved ? saved->h_blocks : nullptr;
    sa.z_blocks = saved ? saved->z_blocks : nullptr;
    sa.s_first = saved ? saved->qat_s_first : nullptr;
    sa.q = (const float*)q;
    sa.k = (const float*)k;
    sa.v = (const float*)v;
    sa.phik = (const float*)w.phik;
    if (g.bf16) {
        sa.tm_q = &mq;
        sa.tm_k = &mk;
        sa.tm_v = &mv;
        sa.tm_phik = &mphi;
        sa.tm_ht = &mht;
        sa.tm_phiq = w.phiq ? &mpq : nullptr;
        sa.phiq = w.phiq;
        sa.tm_out = &mo;
        sa.ol = w.ol;
        if (g.quant) {
            // INT8 QAT (QuantConfig, quant.hpp:15-19): per-tile codes + scales, then the kind::i8 kernel
            if (kc_ready) {  // every code was made on the side stream
                SLA2_CUDA_TRY(cudaStreamWaitEvent(st, kc_ready, 0));
            } else if (plan.qv_codes) {  // Q / V codes are being made beside the router: K~ codes (need mu) only
                SLA2_CUDA_TRY(launch_quant_prep(quant_launch(p, g, w, q, k, v, 2), st, &g_launches));
                SLA2_CUDA_TRY(cudaStreamWaitEvent(st, plan.qv_codes, 0));
            } else {
                SLA2_CUDA_TRY(launch_quant_prep(quant_launch(p, g, w, q, k, v, 1 | 2 | 4), st, &g_launches));
            }
            // the INT8 kernel addresses its bf16 tiles with 2-D [B*H*N][d] maps (N divisible)
            CUtensorMap mq2, mv2, mphi2;
            if (!make_map(&mq2, q, rows, g.d, 64, 64, 2) || !make_map(&mv2, v, rows, g.d, 64, 64, 2) ||
                !make_map(&mphi2, w.phik, rows, g.d, 64, 64, 2))
                return fail(SLA2_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
            sa.tm_q = &mq2;
            sa.tm_v = &mv2;
            sa.tm_phik = &mphi2;
            CUtensorMap mqc, mkc, mvc;
            if (!make_map(&mqc, w.qc, rows, g.d, 128, 128, 1) || !make_map(&mkc, w.kc, rows, g.d, 128, 64, 1) ||
                !make_map(&mvc, w.vct, rows, g.d, 128, 64, 1))
                return fail(SLA2_CUDA_ERROR, "cuTensorMapEncodeTiled failed (int8 codes)");
            SparseI8Launch ia{};
            ia.s = sa;
            ia.qs = w.qs;
            ia.ks = w.ks;
            ia.vs = w.vs;
            ia.tm_qc = &mqc;
            ia.tm_kc = &mkc;
            ia.tm_vct = &mvc;
            if (attn_i8_eligible(ia))
                SLA2_CUDA_TRY(launch_attn_i8(ia, &mphi, &mv, st, &g_launches));
            else
                SLA2_CUDA_TRY(launch_sparse_i8(ia, st, &g_launches));
        } else if (g.fp8) {
            // FP8 P/V (tolerance mode): the persistent kernel with E4M3 P, V and phi(K~)
            CUtensorMap mv8, mphi8;
            if (!make_map3(&mv8, w.v8, (uint64_t)g.BH, (uint64_t)g.N, g.d, 128, 64, 1) ||
                !make_map3(&mphi8, w.phi8, (uint64_t)g.BH, (uint64_t)g.N, g.d, 128, 64, 1))
                return fail(SLA2_CUDA_ERROR, "cuTensorMapEncodeTiled failed (fp8 operands)");
            if (plan.fp8_v) SLA2_CUDA_TRY(cudaStreamWaitEvent(st, plan.fp8_v, 0));
            sa.vamax = w.vamax;
            sa.tm_v8 = &mv8;
            sa.tm_phi8 = &mphi8;
            if (!sparse_v2_eligible(sa))
                return fail(SLA2_CONTRACT_ERROR, "FP8 P/V mode computes out only (no saved state)");
            SLA2_CUDA_TRY(launch_sparse_v2(sa, st, &g_launches));
        } else if (sparse_v2_eligible(sa)) {
            SLA2_CUDA_TRY(launch_sparse_v2(sa, st, &g_launches));
        } else {
            SLA2_CUDA_TRY(launch_sparse_bf16(sa, st, &g_launches));
        }
    } else {
        SLA2_CUDA_TRY(launch_sparse_f32(sa, st, &g_launches));
    }
    if (saved && saved->q_phi)
        SLA2_CUDA_TRY(launch_phi_exact(q, g.bf16, nullptr, saved->q_phi, g.BH * g.N, (int)g.N, (int)g.d, st,
                                       &g_launches));
    if (saved && saved->k_phi)
        SLA2_CUDA_TRY(launch_phi_exact(k, g.bf16, p->smooth ? w.mu : nullptr, saved->k_phi, g.BH * g.N, (int)g.N,
                                       (int)g.d, st, &g_launches));
    return SLA2_OK;
}

// The saved-state members each path can fill (sla2_fwd_saved).
static sla2_status check_saved(const sla2_fwd_params* p, const sla2_fwd_saved* saved) {
    if (!saved) return SLA2_OK;
    if (saved->o_l && !saved->o_s) return fail(SLA2_CONTRACT_ERROR, "saved: o_l requires o_s");
    if ((saved->h_blocks == nullptr) != (saved->z_blocks == nullptr))
        return fail(SLA2_CONTRACT_ERROR, "saved: h_blocks and z_blocks go together");
    if (saved->qat_s_first && p->quant != SLA2_QUANT_INT8)
        return fail(SLA2_CONTRACT_ERROR, "saved: qat_s_first is the INT8 QAT path's hook");
    return SLA2_OK;
}

// Router launch description shared by sla2_router and sla2_forward.
static void fill_router(const sla2_fwd_params* p, const Geo& g, const Workspace& w, const void* q, const void* k,
                        const float* proj_q, const float* proj_k, float* pc_out, uint8_t* mask_out, int32_t* idx,
                        CUtensorMap* mcol, RouterLaunch* ra) {
    *ra = RouterLaunch{};
    ra->q = q;
    ra->k = k;
    ra->bf16 = g.bf16;
    ra->B = g.B;
    ra->H = g.H;
    ra->N = (int)g.N;
    ra->d = (int)g.d;
    ra->bq = (int)g.bq;
    ra->bk = (int)g.bk;
    ra->kappa = (int)g.kappa;
    ra->smooth = p->smooth;
    ra->exact_mu = p->exact_mu;
    ra->inv_sqrt_d = inv_sqrt(g.d);
    ra->proj_q = proj_q;
    ra->proj_k = proj_k;
    ra->tm_kcol = colmean_map(mcol, k, g.bf16, g.BH, g.N, g.d);
    ra->mu_out = w.mu;
    ra->mu_part = w.mu_part;
    ra->qp = w.qp;
    ra->kp = w.kp;
    ra->qbar = w.qbar;
    ra->kbar = w.kbar;
    ra->pc_out = pc_out;
    ra->mask_out = mask_out;
    ra->idx_out = idx ? idx : w.idx;
}

sla2_status sla2_router(const sla2_fwd_params* p, const void* q, const void* k, const float* proj_q,
                        const float* proj_k, float* pc_out, uint8_t* mask_out, int32_t* kv_idx_out, void* workspace,
                        size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = check_common(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    const Geo g = geometry(p);
    if (workspace_bytes < carve(g, nullptr, nullptr) || !workspace)
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_workspace_size)");
    if (!q || !k || !proj_q || !proj_k) return fail(SLA2_CONTRACT_ERROR, "NULL input pointer");
    Workspace w;
    carve(g, workspace, &w);
    RouterLaunch ra;
    CUtensorMap mcol;
    fill_router(p, g, w, q, k, proj_q, proj_k, pc_out, mask_out, kv_idx_out, &mcol, &ra);
    ra.mu_ready = g_mu_ready;
    SLA2_CUDA_TRY(launch_router(ra, (cudaStream_t)stream, &g_launches));
    return SLA2_OK;
}

sla2_status sla2_forward(const sla2_fwd_params* p, const void* q, const void* k, const void* v, const float* proj_q,
                         const float* proj_k, const float* rho, void* out, uint8_t* mask_out, int32_t* kv_idx_out,
                         const sla2_fwd_saved* saved, void* workspace, size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = sla2_check_params(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    const Geo g = geometry(p);
    if (!q || !k || !v || !proj_q || !proj_k || !rho || !out)
        return fail(SLA2_CONTRACT_ERROR, "NULL input/output pointer");
    if ((s = check_saved(p, saved)) != SLA2_OK) return s;
    if (workspace_bytes < carve(g, nullptr, nullptr) || !workspace)
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_workspace_size)");
    Workspace w;
    carve(g, workspace, &w);
    int32_t* idx = kv_idx_out ? kv_idx_out : w.idx;
    cudaStream_t st = (cudaStream_t)stream;
    mark(0, st);
    // the linear precompute needs only mu: the router records mu_ready and the precompute
    // forks off it, overlapping the router's key side (pooling, projection, scores, top-k)
    cudaEvent_t ev_mu = aux_event(12);
    if (!ev_mu) return fail(SLA2_CUDA_ERROR, "cudaEventCreate failed");
    if (g.d == 128 && 4 * g.bk * 128 * (g.bf16 ? 2 : 4) <= 200 * 1024) {
        // router front (mu, query side) -> pooled keys -> router back (projection, scores, top-k),
        // with phi(K~), z_j and Htot forked beside the router's back half
        RouterLaunch ra;
        CUtensorMap mcol;
        fill_router(p, g, w, q, k, proj_q, proj_k, nullptr, mask_out, idx, &mcol, &ra);
        ra.kbar_ready = true;
        // phi(Q) on the query side, beside the serial column mean (written by the query pooling).
        // Measured alternatives: phi(Q) on the linear stream (mu 10 us earlier, but the router's
        // back half 18 us later); starting the linear precompute with the call on its own
        // parallel mean (0.649-0.708 vs 0.632 ms: its CTAs hold the SMs the serial column mean
        // and the router need).
        ra.phiq_out = w.phiq;
        LinPlan plan;
        if (g.quant) {
            // QAT: the Q and V codes do not depend on mu; quantize them on a low-priority side
            // stream beside the router (the K~ codes follow mu in run_linear_and_sparse)
            cudaStream_t qs = aux_stream(3, -1);
            cudaEvent_t ev0 = aux_event(13), ev_qv = aux_event(14);
            SLA2_CUDA_TRY(cudaEventRecord(ev0, st));
            SLA2_CUDA_TRY(cudaStreamWaitEvent(qs, ev0, 0));
            QuantLaunch qa{};
            qa.B = g.B;
            qa.H = g.H;
            qa.N = (int)g.N;
            qa.d = (int)g.d;
            qa.bq = (int)g.bq;
            qa.bk = (int)g.bk;
            qa.tm = (int)g.tm;
            qa.tn = (int)g.tn;
            qa.q = q;
            qa.k = k;
            qa.v = v;
            qa.qc = w.qc;
            qa.qs = w.qs;
            qa.kc = w.kc;
            qa.ks = w.ks;
            qa.vct = w.vct;
            qa.vs = w.vs;
            qa.which = 1 | 4;
            SLA2_CUDA_TRY(launch_quant_prep(qa, qs, &g_launches));
            SLA2_CUDA_TRY(cudaEventRecord(ev_qv, qs));
            plan.qv_codes = ev_qv;
        } else if (g.fp8) {
            // FP8 P/V: V's per-head scale and E4M3 codes do not depend on mu either: a low-priority
            // side stream makes them while the serial column mean holds a few SMs (measured at
            // cfg3fp8: 0.591-0.598 ms; after the linear precompute instead: 0.597-0.600 ms)
            cudaStream_t qs = aux_stream(3, -1);
            cudaEvent_t ev0 = aux_event(13), ev_v = aux_event(14);
            SLA2_CUDA_TRY(cudaEventRecord(ev0, st));
            SLA2_CUDA_TRY(cudaStreamWaitEvent(qs, ev0, 0));
            SLA2_CUDA_TRY(launch_fp8pv_prep(v, nullptr, w.v8, w.phi8, w.vamax, g.BH, g.N, qs, &g_launches));
            SLA2_CUDA_TRY(cudaEventRecord(ev_v, qs));
            plan.fp8_v = ev_v;
        }
        SLA2_CUDA_TRY(launch_router_front(ra, st, &g_launches));
        plan.kprep = true;
        plan.phiq_ready = w.phiq != nullptr;
        plan.kbar = w.kbar;
        plan.between = [&](cudaStream_t rs) -> sla2_status {
            SLA2_CUDA_TRY(launch_router_back(ra, rs, &g_launches));
            return SLA2_OK;
        };
        s = run_linear_and_sparse(p, g, w, q, k, v, rho, idx, nullptr, (int)g.kappa, out, saved, st, plan);
        mark(3, st);
        return s;
    }
    if (p->smooth) {
        g_mu_ready = ev_mu;
    } else if (cudaEventRecord(ev_mu, st) != cudaSuccess) {  // phi(K) on raw K: fork at once
        return fail(SLA2_CUDA_ERROR, "cudaEventRecord failed");
    }
    s = sla2_router(p, q, k, proj_q, proj_k, nullptr, mask_out, idx, workspace, workspace_bytes, stream);
    g_mu_ready = nullptr;
    const int router_launches = g_launches;
    if (s != SLA2_OK) return s;
    LinPlan plan;
    plan.dep = ev_mu;
    s = run_linear_and_sparse(p, g, w, q, k, v, rho, idx, nullptr, (int)g.kappa, out, saved, st, plan);
    mark(3, st);
    g_launches += router_launches;
    return s;
}

sla2_status sla2_smooth_k(const sla2_fwd_params* p, const void* k, float* mean_out, float* ktilde_out, void* stream) {
    g_launches = 0;
    sla2_status s = check_common(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    if (!k || !mean_out) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    if (ktilde_out) return fail(SLA2_CONTRACT_ERROR, "ktilde_out is not supported; pass NULL");
    CUtensorMap mcol;
    const bool bf = p->dtype == SLA2_BF16;
    SLA2_CUDA_TRY(launch_colmean(k, colmean_map(&mcol, k, bf, p->B * p->H, p->N, p->d), bf, mean_out,
                                 (int)(p->B * p->H), (int)p->N, (int)p->d, (cudaStream_t)stream, &g_launches));
    return SLA2_OK;
}

sla2_status sla2_quantize(const sla2_fwd_params* p, const void* q, const void* k, const void* v, int8_t* q_codes,
                          float* q_scales, int8_t* k_codes, float* k_scales, int8_t* v_codes, float* v_scales,
                          void* workspace, size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = sla2_check_params(p);
    if (s != SLA2_OK) return s;
    if (p->dtype != SLA2_BF16 || p->quant != SLA2_QUANT_INT8)
        return fail(SLA2_CONTRACT_ERROR, "sla2_quantize: the INT8 QAT path (dtype bf16, quant int8)");
    if ((s = check_device()) != SLA2_OK) return s;
    if (!q || !k || !v || !q_codes || !q_scales || !k_codes || !k_scales || !v_codes || !v_scales)
        return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    if (workspace_bytes < carve(g, nullptr, nullptr) || !workspace)
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_workspace_size)");
    Workspace w;
    carve(g, workspace, &w);
    cudaStream_t st = (cudaStream_t)stream;
    CUtensorMap mcol;
    if (p->smooth)  // K~ = K - mu with the reference's serial mean (quant.hpp:88-96)
        SLA2_CUDA_TRY(launch_colmean(k, colmean_map(&mcol, k, true, g.BH, g.N, g.d), true, w.mu, (int)g.BH, (int)g.N,
                                     (int)g.d, st, &g_launches));
    QuantLaunch qa{};
    qa.B = g.B;
    qa.H = g.H;
    qa.N = (int)g.N;
    qa.d = (int)g.d;
    qa.bq = (int)g.bq;
    qa.bk = (int)g.bk;
    qa.tm = (int)g.tm;
    qa.tn = (int)g.tn;
    qa.q = q;
    qa.k = k;
    qa.v = v;
    qa.mu = w.mu;
    qa.smooth = p->smooth;
    qa.qc = q_codes;
    qa.qs = q_scales;
    qa.kc = k_codes;
    qa.ks = k_scales;
    qa.vct = v_codes;
    qa.vs = v_scales;
    SLA2_CUDA_TRY(launch_quant_prep(qa, st, &g_launches));
    return SLA2_OK;
}

sla2_status sla2_linear_precompute(const sla2_fwd_params* p, const void* k, const void* v, float* k_phi_out,
                                   float* z_blocks_out, float* h_total_out, float* z_total_out, void* workspace,
                                   size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = sla2_check_params(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    if (!k || !v) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    if (workspace_bytes < carve(g, nullptr, nullptr) || !workspace)
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_workspace_size)");
    Workspace w;
    carve(g, workspace, &w);
    cudaStream_t st = (cudaStream_t)stream;
    CUtensorMap mcol, mk, mv, mphi;
    if (p->smooth)  // the exact serial mean (quant.hpp:88-96), as the forward uses
        SLA2_CUDA_TRY(launch_colmean(k, colmean_map(&mcol, k, g.bf16, g.BH, g.N, g.d), g.bf16, w.mu, (int)g.BH,
                                     (int)g.N, (int)g.d, st, &g_launches));
    LinearLaunch la{};
    la.k = k;
    la.v = v;
    la.bf16 = g.bf16;
    la.BH = g.BH;
    la.N = (int)g.N;
    la.d = (int)g.d;
    la.bk = (int)g.bk;
    la.mu = p->smooth ? w.mu : nullptr;
    la.phik = w.phik;
    la.zblk = w.zblk;
    la.ztot = w.ztot;
    la.hpart = w.hpart;
    la.htot = w.htot;
    la.htot16 = w.htot16;
    la.nchunk = g.nchunk;
    if (g.bf16) {
        const uint64_t BH = (uint64_t)g.BH, N = (uint64_t)g.N;
        if (!make_map3(&mk, k, BH, N, g.d, 64, 64, 2) || !make_map3(&mv, v, BH, N, g.d, 64, 64, 2) ||
            !make_map3(&mphi, w.phik, BH, N, g.d, 64, 64, 2))
            return fail(SLA2_CUDA_ERROR, "cuTensorMapEncodeTiled failed (pointers must be 16-byte aligned)");
        la.tm_k = &mk;
        la.tm_v = &mv;
        la.tm_phik = &mphi;
    }
    SLA2_CUDA_TRY(launch_linear_prep(la, st, &g_launches));
    const size_t dd = (size_t)(g.d * g.d) * 4;
    if (z_blocks_out)
        SLA2_CUDA_TRY(cudaMemcpyAsync(z_blocks_out, w.zblk, (size_t)(g.BH * g.tn * g.d) * 4, cudaMemcpyDeviceToDevice, st));
    if (h_total_out) SLA2_CUDA_TRY(cudaMemcpyAsync(h_total_out, w.htot, (size_t)g.BH * dd, cudaMemcpyDeviceToDevice, st));
    if (z_total_out)
        SLA2_CUDA_TRY(cudaMemcpyAsync(z_total_out, w.ztot, (size_t)(g.BH * g.d) * 4, cudaMemcpyDeviceToDevice, st));
    if (k_phi_out)
        SLA2_CUDA_TRY(launch_phi_exact(k, g.bf16, p->smooth ? w.mu : nullptr, k_phi_out, g.BH * g.N, (int)g.N, (int)g.d,
                                       st, &g_launches));
    return SLA2_OK;
}

sla2_status sla2_hard_topk(const sla2_fwd_params* p, const float* pc, uint8_t* mask_out, int32_t* kv_idx_out,
                           void* stream) {
    g_launches = 0;
    g_last_error.clear();
    // only the score-matrix geometry matters here: rows tm = N / bq, columns tn = N / bk
    if (!p) return fail(SLA2_CONTRACT_ERROR, "params is NULL");
    if (p->B <= 0 || p->H <= 0 || p->N <= 0 || p->bq <= 0 || p->bk <= 0 || p->N % p->bq || p->N % p->bk)
        return fail(SLA2_SHAPE_ERROR, "hard_topk: bad score-matrix geometry");
    if (!(p->k_percent > 0.0 && p->k_percent <= 100.0))
        return fail(SLA2_SHAPE_ERROR, "hard_topk: k_percent must be in (0, 100]");  // router.hpp:108-110
    sla2_status s = check_device();
    if (s != SLA2_OK) return s;
    if (!pc || !kv_idx_out) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    SLA2_CUDA_TRY(launch_topk_only(pc, (int)g.BH, (int)g.tm, (int)g.tn, (int)g.kappa, mask_out, kv_idx_out,
                                   (cudaStream_t)stream, &g_launches));
    return SLA2_OK;
}

sla2_status sla2_sparse_fwd(const sla2_fwd_params* p, const void* q, const void* k, const void* v, const float* rho,
                            const uint8_t* mask, void* out, const sla2_fwd_saved* saved, void* workspace,
                            size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = sla2_check_params(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    const Geo g = geometry(p);
    if (!q || !k || !v || !rho || !mask || !out) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    if ((s = check_saved(p, saved)) != SLA2_OK) return s;
    if (workspace_bytes < carve(g, nullptr, nullptr) || !workspace)
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_workspace_size)");
    Workspace w;
    carve(g, workspace, &w);
    cudaStream_t st = (cudaStream_t)stream;
    SLA2_CUDA_TRY(cudaMemsetAsync(w.flag, 0, sizeof(int), st));
    SLA2_CUDA_TRY(launch_mask_to_idx(mask, (int)(g.BH * g.tm), (int)g.tn, w.idx, w.cnt, w.flag, st, &g_launches));
    int flag = 0;
    SLA2_CUDA_TRY(cudaMemcpyAsync(&flag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    SLA2_CUDA_TRY(cudaStreamSynchronize(st));
    if (flag) return fail(SLA2_SHAPE_ERROR, "sla2_forward_blockwise: mask row keeps no blocks");  // attention.hpp:445
    CUtensorMap mcol;
    if (p->smooth)
        SLA2_CUDA_TRY(launch_colmean(k, colmean_map(&mcol, k, g.bf16, g.BH, g.N, g.d), g.bf16, w.mu, (int)g.BH,
                                     (int)g.N, (int)g.d, st, &g_launches));
    const int ml = g_launches;
    s = run_linear_and_sparse(p, g, w, q, k, v, rho, w.idx, w.cnt, (int)g.tn, out, saved, st);
    g_launches += ml;
    return s;
}

sla2_status sla2_dense_fwd(const sla2_fwd_params* p, const void* q, const void* k, const void* v, void* out,
                           void* workspace, size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = sla2_check_params(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    if (p->dtype != SLA2_BF16) return fail(SLA2_CONTRACT_ERROR, "sla2_dense_fwd is the bf16 tcgen05 baseline");
    const Geo g = geometry(p);
    if (!q || !k || !v || !out) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    (void)workspace;
    (void)workspace_bytes;
    CUtensorMap mq, mk, mv;
    const uint64_t rows = (uint64_t)(g.BH * g.N);
    CUtensorMap mo;
    (void)rows;
    const uint64_t BH = (uint64_t)g.BH, N = (uint64_t)g.N;
    if (!make_map3(&mq, q, BH, N, g.d, 64, 64, 2) || !make_map3(&mk, k, BH, N, g.d, 64, 64, 2) ||
        !make_map3(&mv, v, BH, N, g.d, 64, 64, 2) || !make_map3(&mo, out, BH, N, g.d, 64, 64, 2))
        return fail(SLA2_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    SparseLaunch sa{};
    sa.B = g.B;
    sa.H = g.H;
    sa.N = (int)g.N;
    sa.d = (int)g.d;
    sa.bq = (int)g.bq;
    sa.bk = (int)g.bk;
    sa.tm = (int)g.tm;
    sa.tn = (int)g.tn;
    sa.kstride = (int)g.tn;
    sa.kappa = (int)g.tn;
    sa.dense = 1;
    sa.inv_sqrt_d = inv_sqrt(g.d);
    sa.out = out;
    sa.tm_q = &mq;
    sa.tm_k = &mk;
    sa.tm_v = &mv;
    sa.tm_phik = &mk;
    sa.tm_out = &mo;
    if (sparse_fa_eligible(sa)) {  // the two-query-block tcgen05 attention kernel (sparse_fa.cu)
        SLA2_CUDA_TRY(launch_sparse_fa(sa, (cudaStream_t)stream, &g_launches));
        return SLA2_OK;
    }
    SLA2_CUDA_TRY(launch_sparse_bf16(sa, (cudaStream_t)stream, &g_launches));
    return SLA2_OK;
}

// ---------------------------------------------------------------- backward (attention.hpp:610-809)
static sla2_status check_backward(const sla2_fwd_params* p) {
    sla2_status s = check_common(p);
    if (s != SLA2_OK) return s;
    if (p->dtype != SLA2_F32)
        return fail(SLA2_CONTRACT_ERROR, "sla2_backward: fp32 tensors (the backward is full precision, SPEC.md:358)");
    if (p->N % p->bq != 0 || p->N % p->bk != 0)
        return fail(SLA2_SHAPE_ERROR, "AttentionInputs: N must be divisible by bq and bk");  // attention.hpp:39-41
    if (p->d > 128 || p->bk > 64 || (p->bq > 64 && (p->bq % 64 != 0 || (p->d > 64 && p->bq > 128))) ||
        p->N / p->bq > 1024)
        return fail(SLA2_CONTRACT_ERROR,
                    "sla2_backward: d <= 128, bk <= 64, bq <= 64 or a multiple of 64 (<= 128 when d > 64), tm <= 1024");
    return SLA2_OK;
}

static size_t carve_backward(const Geo& g, void* base, BackwardLaunch* a) {
    Carver c{reinterpret_cast<uint8_t*>(base)};
    BackwardLaunch t{};
    t.mu = c.take<float>(g.BH * g.d);
    t.phik = c.take<float>(g.BH * g.N * g.d);
    t.h = c.take<float>(g.BH * g.tn * g.d * g.d);
    t.z = c.take<float>(g.BH * g.tn * g.d);
    t.htot = c.take<float>(g.BH * g.d * g.d);
    t.ztot = c.take<float>(g.BH * g.d);
    t.dh = c.take<float>(g.BH * g.tm * g.d * g.d);
    t.dz = c.take<float>(g.BH * g.tm * g.d);
    t.dsr = c.take<float>(g.BH * g.N);
    if (a) {
        a->mu = t.mu; a->phik = t.phik; a->h = t.h; a->z = t.z; a->htot = t.htot; a->ztot = t.ztot;
        a->dh = t.dh; a->dz = t.dz; a->dsr = t.dsr;
    }
    return c.off + 256;
}

size_t sla2_backward_workspace_size(const sla2_fwd_params* p) {
    if (check_backward(p) != SLA2_OK) return 0;
    return carve_backward(geometry(p), nullptr, nullptr);
}

sla2_status sla2_backward(const sla2_fwd_params* p, const void* q, const void* k, const void* v, const float* rho,
                          const uint8_t* mask, const float* o_s, const float* o_l, const float* big_l,
                          const void* d_out, void* dq, void* dk, void* dv, float* drho, void* workspace,
                          size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = check_backward(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    if (!q || !k || !v || !rho || !mask || !o_s || !o_l || !big_l || !d_out || !dq || !dk || !dv || !drho)
        return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    if (!workspace || workspace_bytes < carve_backward(g, nullptr, nullptr))
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_backward_workspace_size)");
    cudaStream_t st = (cudaStream_t)stream;
    // every row keeps a block (the forward's own precondition, attention.hpp:442-447)
    CUtensorMap unused;
    (void)unused;
    BackwardLaunch a{};
    carve_backward(g, workspace, &a);
    a.BH = g.BH;
    a.H = g.H;
    a.N = (int)g.N;
    a.d = (int)g.d;
    a.bq = (int)g.bq;
    a.bk = (int)g.bk;
    a.tm = (int)g.tm;
    a.tn = (int)g.tn;
    a.smooth = p->smooth;
    a.inv_sqrt_d = inv_sqrt(g.d);
    a.q = (const float*)q;
    a.k = (const float*)k;
    a.v = (const float*)v;
    a.d_out = (const float*)d_out;
    a.o_s = o_s;
    a.o_l = o_l;
    a.big_l = big_l;
    a.rho = rho;
    a.mask = mask;
    a.dq = (float*)dq;
    a.dk = (float*)dk;
    a.dv = (float*)dv;
    a.drho = drho;
    SLA2_CUDA_TRY(launch_backward(a, st, &g_launches));
    return SLA2_OK;
}

// ---------------------------------------------------------------- stage-1 soft routing
// soft_topk (router.hpp:126-190) and sla2_forward_blockwise with a SoftMask (attention.hpp:484-558)
static sla2_status check_soft(const sla2_fwd_params* p, const char* who) {
    sla2_status s = check_common(p);
    if (s != SLA2_OK) return s;
    if (p->dtype != SLA2_F32 || p->quant != SLA2_QUANT_NONE)
        return fail(SLA2_CONTRACT_ERROR, std::string(who) + ": fp32 without quantization (the stage-1 training path)");
    if (p->N % p->bq != 0 || p->N % p->bk != 0)
        return fail(SLA2_SHAPE_ERROR, "AttentionInputs: N must be divisible by bq and bk");  // attention.hpp:39-41
    if (p->d > 64 || p->bq > 64 || p->bk > 64)
        return fail(SLA2_CONTRACT_ERROR, std::string(who) + ": d, bq, bk <= 64 on this path");
    return SLA2_OK;
}

sla2_status sla2_soft_topk(const sla2_fwd_params* p, const float* pc, float* values, float* lambdas, void* stream) {
    g_launches = 0;
    // only the score geometry tm x tn matters here; soft_topk clamps any k% through topk_budget
    // (router.hpp:130-134) instead of hard_topk's (0, 100] check
    sla2_status s = check_common(p, false);
    if (s != SLA2_OK) return s;
    if (p->N % p->bq != 0 || p->N % p->bk != 0)
        return fail(SLA2_SHAPE_ERROR, "AttentionInputs: N must be divisible by bq and bk");
    if ((s = check_device()) != SLA2_OK) return s;
    if (!pc || !values || !lambdas) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    cudaStream_t st = (cudaStream_t)stream;
    // per-device flag (a process may drive several GPUs)
    thread_local std::unordered_map<int, int*> dfails;
    int dev = 0;
    SLA2_CUDA_TRY(cudaGetDevice(&dev));
    int*& dfail = dfails[dev];
    if (!dfail) SLA2_CUDA_TRY(cudaMalloc(&dfail, sizeof(int)));
    SLA2_CUDA_TRY(cudaMemsetAsync(dfail, 0, sizeof(int), st));
    const double kappa = (double)sla2_topk_budget(p->k_percent, g.tn);
    SLA2_CUDA_TRY(launch_soft_topk(pc, (int)(g.BH * g.tm), (int)g.tn, kappa, (double)p->tau, values, lambdas, dfail,
                                   st, &g_launches));
    int hfail = 0;  // the reference throws on a row that does not converge: one D2H read
    SLA2_CUDA_TRY(cudaMemcpyAsync(&hfail, dfail, sizeof(int), cudaMemcpyDeviceToHost, st));
    SLA2_CUDA_TRY(cudaStreamSynchronize(st));
    if (hfail) return fail(SLA2_NUMERIC_ERROR, "soft_topk: bisection did not converge");
    return SLA2_OK;
}

sla2_status sla2_soft_topk_backward(const sla2_fwd_params* p, const float* values, const float* upstream,
                                    float* grad, void* stream) {
    g_launches = 0;
    sla2_status s = check_common(p);  // the score geometry tm x tn and tau (> 0)
    if (s != SLA2_OK) return s;
    if (p->N % p->bq != 0 || p->N % p->bk != 0)
        return fail(SLA2_SHAPE_ERROR, "AttentionInputs: N must be divisible by bq and bk");
    if ((s = check_device()) != SLA2_OK) return s;
    if (!values || !upstream || !grad) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    const float inv_tau = 1.0f / p->tau;  // T(1) / softmask.tau in float (router.hpp:206)
    SLA2_CUDA_TRY(launch_soft_topk_backward(values, upstream, grad, g.BH * g.tm * g.tn, inv_tau,
                                            (cudaStream_t)stream, &g_launches));
    return SLA2_OK;
}

static size_t carve_soft(const Geo& g, void* base, SoftLaunch* a, float** mu, float** phik) {
    Carver c{reinterpret_cast<uint8_t*>(base)};
    float* m = c.take<float>(g.BH * g.d);
    float* pk = c.take<float>(g.BH * g.N * g.d);
    float* h = c.take<float>(g.BH * g.tn * g.d * g.d);
    float* z = c.take<float>(g.BH * g.tn * g.d);
    if (a) {
        *mu = m;
        *phik = pk;
        a->h = h;
        a->z = z;
    }
    return c.off + 256;
}

size_t sla2_forward_soft_workspace_size(const sla2_fwd_params* p) {
    if (check_soft(p, "sla2_forward_soft") != SLA2_OK) return 0;
    return carve_soft(geometry(p), nullptr, nullptr, nullptr, nullptr);
}

sla2_status sla2_forward_soft(const sla2_fwd_params* p, const void* q, const void* k, const void* v, const float* rho,
                              const float* values, void* out, const sla2_fwd_saved* saved, void* workspace,
                              size_t workspace_bytes, void* stream) {
    g_launches = 0;
    sla2_status s = check_soft(p, "sla2_forward_soft");
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    if (!q || !k || !v || !rho || !values || !out) return fail(SLA2_CONTRACT_ERROR, "NULL pointer");
    const Geo g = geometry(p);
    if (!workspace || workspace_bytes < carve_soft(g, nullptr, nullptr, nullptr, nullptr))
        return fail(SLA2_CONTRACT_ERROR, "workspace too small (see sla2_forward_soft_workspace_size)");
    cudaStream_t st = (cudaStream_t)stream;
    SoftLaunch a{};
    float *mu = nullptr, *phik = nullptr;
    carve_soft(g, workspace, &a, &mu, &phik);
    if (p->smooth) SLA2_CUDA_TRY(launch_colmean(k, nullptr, false, mu, (int)g.BH, (int)g.N, (int)g.d, st, &g_launches));
    a.BH = g.BH;
    a.H = g.H;
    a.N = (int)g.N;
    a.d = (int)g.d;
    a.bq = (int)g.bq;
    a.bk = (int)g.bk;
    a.tm = (int)g.tm;
    a.tn = (int)g.tn;
    a.inv_sqrt_d = inv_sqrt(g.d);
    a.q = (const float*)q;
    a.k = (const float*)k;
    a.v = (const float*)v;
    a.mu = p->smooth ? mu : nullptr;
    a.values = values;
    a.rho = rho;
    a.out = (float*)out;
    a.o_s = saved ? saved->o_s : nullptr;
    a.o_l = saved ? saved->o_l : nullptr;
    a.big_l = saved ? saved->big_l : nullptr;
    SLA2_CUDA_TRY(launch_keyblock_linear(a.k, a.v, a.mu, phik, const_cast<float*>(a.h), const_cast<float*>(a.z), g.BH,
                                         a.N, a.d, a.bk, st, &g_launches));
    SLA2_CUDA_TRY(launch_soft_forward(a, st, &g_launches));
    return SLA2_OK;
}

sla2_status sla2_forward_host(const sla2_fwd_params* p, const void* q, const void* k, const void* v,
                              const float* proj_q, const float* proj_k, const float* rho, void* out,
                              uint8_t* mask_out) {
    sla2_status s = sla2_check_params(p);
    if (s != SLA2_OK) return s;
    if ((s = check_device()) != SLA2_OK) return s;
    if (!q || !k || !v || !proj_q || !proj_k || !rho || !out)
        return fail(SLA2_CONTRACT_ERROR, "NULL input/output pointer");
    // Every (b, h) slice is independent, so the call is pipelined per head: the
    // copy engine brings head c+1 in while head c computes and head c-1 goes back out.
    // PCIe, not the GPU, bounds this path; the pipeline hides the compute and the D2H tail.
    const Geo g = geometry(p);
    const size_t esz = g.bf16 ? 2 : 4;
    const size_t head = (size_t)(g.N * g.d) * esz;
    const size_t tensor = (size_t)g.BH * head;
    const size_t projb = (size_t)(g.H * g.d * g.d) * 4, rhob = (size_t)(g.H * g.tm) * 4;
    const size_t head_mask = (size_t)(g.tm * g.tn), maskb = (size_t)g.BH * head_mask;
    sla2_fwd_params hp = *p;  // one head per call
    hp.B = 1;
    hp.H = 1;
    const size_t wsb = carve(geometry(&hp), nullptr, nullptr);
    // one cached device arena and three streams per (thread, device). One upload stream: a
    // second one (a head's V beside its K and Q) measured slower, 7.08 vs 6.70 ms at cfg2 -- the
    // copies already run at the link's rate (~45 GB/s pinned H2D on the box; tools/e2e_ab.py)
    int dev = 0;
    SLA2_CUDA_TRY(cudaGetDevice(&dev));
    struct Arena {
        void* ptr = nullptr;
        size_t bytes = 0;
    };
    thread_local std::unordered_map<int, Arena> arenas;
    Arena& ar = arenas[dev];
    const size_t need = 4 * tensor + 2 * projb + rhob + maskb + wsb + 10 * 256;
    if (need > ar.bytes) {
        if (ar.ptr) cudaFree(ar.ptr);
        ar.ptr = nullptr;
        ar.bytes = 0;
        SLA2_CUDA_TRY(cudaMalloc(&ar.ptr, need));
        ar.bytes = need;
    }
    void* arena = ar.ptr;
    cudaStream_t st = aux_stream(20, 0), up = aux_stream(21, 0), down = aux_stream(22, 0);
    cudaEvent_t ev_in = aux_event(20), ev_out = aux_event(21);
    if (!st || !up || !down || !ev_in || !ev_out) return fail(SLA2_CUDA_ERROR, "stream/event creation failed");
    Carver c{reinterpret_cast<uint8_t*>(arena)};
    uint8_t* dq = c.take<uint8_t>(tensor);
    uint8_t* dk = c.take<uint8_t>(tensor);
    uint8_t* dv = c.take<uint8_t>(tensor);
    uint8_t* dout = c.take<uint8_t>(tensor);
    float* dpq = c.take<float>(projb / 4);
    float* dpk = c.take<float>(projb / 4);
    float* drho = c.take<float>(rhob / 4);
    uint8_t* dmask = c.take<uint8_t>(maskb);
    void* dws = c.take<uint8_t>(wsb);
    const uint8_t *hq = static_cast<const uint8_t*>(q), *hk = static_cast<const uint8_t*>(k),
                  *hv = static_cast<const uint8_t*>(v);
    SLA2_CUDA_TRY(cudaMemcpyAsync(dpq, proj_q, projb, cudaMemcpyHostToDevice, up));
    SLA2_CUDA_TRY(cudaMemcpyAsync(dpk, proj_k, projb, cudaMemcpyHostToDevice, up));
    SLA2_CUDA_TRY(cudaMemcpyAsync(drho, rho, rhob, cudaMemcpyHostToDevice, up));
    int launches = 0;
    for (int64_t bh = 0; bh < g.BH; ++bh) {
        const size_t o = (size_t)bh * head;
        const int64_t h = bh % g.H;
        // K first: the column mean, the head's latency-bound first stage, needs only K
        SLA2_CUDA_TRY(cudaMemcpyAsync(dk + o, hk + o, head, cudaMemcpyHostToDevice, up));
        SLA2_CUDA_TRY(cudaMemcpyAsync(dq + o, hq + o, head, cudaMemcpyHostToDevice, up));
        SLA2_CUDA_TRY(cudaMemcpyAsync(dv + o, hv + o, head, cudaMemcpyHostToDevice, up));
        SLA2_CUDA_TRY(cudaEventRecord(ev_in, up));
        SLA2_CUDA_TRY(cudaStreamWaitEvent(st, ev_in, 0));
        uint8_t* hm = mask_out ? dmask + (size_t)bh * head_mask : nullptr;
        s = sla2_forward(&hp, dq + o, dk + o, dv + o, dpq + h * g.d * g.d, dpk + h * g.d * g.d, drho + h * g.tm,
                         dout + o, hm, nullptr, nullptr, dws, wsb, st);
        if (s != SLA2_OK) {
            cudaStreamSynchronize(st);
            return s;
        }
        launches += g_launches;
        SLA2_CUDA_TRY(cudaEventRecord(ev_out, st));
        SLA2_CUDA_TRY(cudaStreamWaitEvent(down, ev_out, 0));
        SLA2_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(out) + o, dout + o, head, cudaMemcpyDeviceToHost, down));
        if (mask_out)
            SLA2_CUDA_TRY(cudaMemcpyAsync(mask_out + (size_t)bh * head_mask, hm, head_mask, cudaMemcpyDeviceToHost, down));
    }
    g_launches = launches;
    SLA2_CUDA_TRY(cudaStreamSynchronize(down));
    SLA2_CUDA_TRY(cudaStreamSynchronize(st));
    return SLA2_OK;
}

}  // extern "C"
