// mkq_abi.cu -- the C ABI of include/mkq.h: argument validation, TMA
// descriptor encoding/caching, kernel dispatch and the BERT-layer
// orchestration.  Everything here only enqueues work on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "../../include/mkq.h"
#include "attention.cuh"
#include "attention_sm100.cuh"
#include "attention_pp_sm100.cuh"
#include "attention_i8.cuh"
#include "gemm_sm100.cuh"
#include "gemm2_sm100.cuh"
#include "gemm_mma_small.cuh"
#include "requant.cuh"
#include "layernorm.cuh"
#include "quantize.cuh"
#include "qat.cuh"
#include "calib.cuh"

#define MKQ_VERSION 10000

#ifdef MKQ_TTRACE
extern "C" __attribute__((visibility("default"))) int mkq_debug_set_ttrace(void* p) {
    unsigned long long* q = static_cast<unsigned long long*>(p);
    return (int)cudaMemcpyToSymbol(mkq::g_ttrace, &q, sizeof(q));
}
#endif

namespace {

thread_local char g_err[512] = "";

mkq_status fail(mkq_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

mkq_status cuda_fail(cudaError_t e, const char* what) {
    return fail(MKQ_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Launch with programmatic dependent launch (PDL, griddepcontrol in the
// kernels) so a kernel's prologue overlaps the previous kernel's tail; in a
// CUDA graph the attribute becomes a programmatic edge.  MKQ_PDL=0 disables.
bool pdl_enabled() {
    static const bool on = [] { const char* e = getenv("MKQ_PDL"); return !(e && strcmp(e, "0") == 0); }();
    return on;
}

// PDL only for latency-bound problem sizes (<= 8192 token rows): on the
// BERT-large bench layer (131072 rows) it measured 160 us slower per layer
// (2.94 -> 3.10 ms), at 440-2298 tokens ~2 us faster.
thread_local bool t_pdl_rows_ok = true;
struct PdlScope {   // sets the row-count gate for the launches of one API call
    bool prev;
    explicit PdlScope(int64_t rows) : prev(t_pdl_rows_ok) { t_pdl_rows_ok = rows <= 8192; }
    ~PdlScope() { t_pdl_rows_ok = prev; }
};

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (pdl_enabled() && t_pdl_rows_ok) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = (unsigned)cluster;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

bool finite_pos(float s) { return std::isfinite(s) && s > 0.0f; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct DevInfo {
    int ok = -1;
    int sms = 0;
};

std::mutex g_mu;
DevInfo g_dev[64];

mkq_status check_device(int* sms = nullptr) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MKQ_ERR_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
    }
    if (dev < 0 || dev >= 64) return fail(MKQ_ERR_DEVICE, "device ordinal %d", dev);
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo& d = g_dev[dev];
    if (d.ok < 0) {
        int maj = 0, min = 0;
        cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        d.ok = (maj == 10 && min == 0) ? 1 : 0;
        if (!d.ok) snprintf(g_err, sizeof(g_err), "device %d is sm_%d%d, need sm_100 (B200)", dev, maj, min);
    }
    if (!d.ok) return MKQ_ERR_DEVICE;
    if (sms) *sms = d.sms;
    return MKQ_OK;
}

// ------------------------------------------------------------------ TMA maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

using MapKey = std::tuple<uintptr_t, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t, int, int, int>;
std::map<MapKey, CUtensorMap> g_maps;

// 2-D map over a row-major matrix: `inner` elements of `dtype` per row, `rows`
// rows, row stride `ld` bytes; box {box_inner, box_rows}; swizzle mode.
mkq_status make_map_t(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, uint64_t inner, uint64_t rows,
                      uint64_t ld, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swz) {
    int dev = 0;
    cudaGetDevice(&dev);
    MapKey key{reinterpret_cast<uintptr_t>(base), inner, rows, ld, box_inner, box_rows, (int)swz, dev, (int)dtype};
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_maps.find(key);
        if (it != g_maps.end()) {
            *out = it->second;
            return MKQ_OK;
        }
    }
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(MKQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {ld};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(out, dtype, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(MKQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps[key] = *out;
    return MKQ_OK;
}

mkq_status make_map(CUtensorMap* out, const void* base, uint64_t inner, uint64_t rows, uint64_t ld,
                    uint32_t box_inner, uint32_t box_rows, bool swz128) {
    return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_UINT8, inner, rows, ld, box_inner, box_rows,
                      swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
}

// Output map of the 2-CTA epilogue: 32-row blocks (16 columns of 4-byte
// outputs, 32 columns otherwise) staged in shared memory with the swizzle
// matching mkq::stg_off().
mkq_status make_out_map(CUtensorMap* out, void* base, int mode, int64_t M, int64_t N, int64_t ldo) {
    switch (mode) {
    case MKQ_OUT_F32:
        return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, N, M, ldo, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    case MKQ_OUT_I32:
        return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_INT32, N, M, ldo, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    case MKQ_OUT_F16:
        return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, N, M, ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    case MKQ_OUT_BF16:
        return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, N, M, ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    case MKQ_OUT_I8:
        return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_UINT8, N, M, ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_32B);
    default:  // MKQ_OUT_I4: packed bytes
        return make_map_t(out, base, CU_TENSOR_MAP_DATA_TYPE_UINT8, N / 2, M, ldo, 16, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
}

// ------------------------------------------------------------------ GEMM dispatch
template <class Cfg, bool kCl = false>
mkq_status launch_gemm(const void* a, int64_t lda, const void* w, int64_t ldw, int M, int N, int K,
                       const mkq::EpiParams& ep, int sms, cudaStream_t st, int splits = 1) {
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(mkq::gemm_i8tc_kernel<Cfg, kCl>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        attr_set[dev] = true;
    }
    CUtensorMap ma, mb;
    const uint64_t kbytes = Cfg::kInt4 ? (uint64_t)K / 2 : (uint64_t)K;
    const uint32_t box_in = Cfg::kInt4 ? Cfg::BK / 2 : Cfg::BK;
    // kTA (small-M int4): packed 128-byte A rows with the 128-byte swizzle (conflict-free row reads by lane)
    mkq_status s = make_map(&ma, a, kbytes, (uint64_t)M, (uint64_t)lda, box_in, Cfg::BM, !Cfg::kInt4 || Cfg::kTA);
    if (s != MKQ_OK) return s;
    s = make_map(&mb, w, kbytes, (uint64_t)N, (uint64_t)ldw, box_in, Cfg::BN, !Cfg::kInt4 || Cfg::kTA);
    if (s != MKQ_OK) return s;
    const int tiles = ((M + Cfg::BM - 1) / Cfg::BM) * ((N + Cfg::BN - 1) / Cfg::BN);
    // output map: TMA stores of the small-M plan's epilogues (unused otherwise)
    CUtensorMap mo = ma;
    if (kCl) {
        s = make_out_map(&mo, ep.out, ep.mode, M, N, ep.ldo_bytes);
        if (s != MKQ_OK) return s;
    }
    cudaError_t e;
    if constexpr (kCl) {
        // one CTA per (tile, K split); the splits of a tile form one cluster
        e = launch_k(mkq::gemm_i8tc_kernel<Cfg, true>, dim3((unsigned)(tiles * splits)), dim3(Cfg::kThreads),
                     Cfg::kSmem, st, splits, ma, mb, mo, ep, M, N, K, splits);
    } else {
        const int grid = tiles < sms ? tiles : sms;
        e = launch_k(mkq::gemm_i8tc_kernel<Cfg, false>, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, st, 1, ma, mb,
                     mo, ep, M, N, K, 1);
    }
    if (e != cudaSuccess) return cuda_fail(e, "gemm launch");
    return MKQ_OK;
}

bool code_range_ok(int bits, int qmin, int qmax) {
    const int lo = bits == 4 ? -8 : -128, hi = bits == 4 ? 7 : 127;
    return qmin >= lo && qmax <= hi && qmin < qmax;
}

template <class Cfg>
mkq_status launch_gemm2(const void* a, int64_t lda, const void* w, int64_t ldw, int M, int N, int K,
                        const mkq::Epi2Params& ep, int sms, cudaStream_t st) {
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(mkq::gemm_w4a4_2cta_kernel<Cfg>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        attr_set[dev] = true;
    }
    CUtensorMap ma, mb;
    mkq_status s = make_map(&ma, a, (uint64_t)K / 2, (uint64_t)M, (uint64_t)lda, Cfg::BK / 2, Cfg::BM, false);
    if (s != MKQ_OK) return s;
    s = make_map(&mb, w, (uint64_t)K / 2, (uint64_t)N, (uint64_t)ldw, Cfg::BK / 2, Cfg::BNH, false);
    if (s != MKQ_OK) return s;
    CUtensorMap mo;
    s = make_out_map(&mo, ep.e.out, ep.e.mode, M, N, ep.e.ldo_bytes);
    if (s != MKQ_OK) return s;
    const int tiles = ((M + 2 * Cfg::BM - 1) / (2 * Cfg::BM)) * ((N + Cfg::BN - 1) / Cfg::BN);
    static const int max_cl = [] { const char* v = getenv("MKQ_MAX_CLUSTERS"); return v ? atoi(v) : 0; }();
    int clusters = tiles < sms / 2 ? tiles : sms / 2;
    if (max_cl > 0 && clusters > max_cl) clusters = max_cl;
    cudaError_t e = launch_k(mkq::gemm_w4a4_2cta_kernel<Cfg>, dim3(2 * clusters), dim3(Cfg::kThreads), Cfg::kSmem,
                             st, 1, ma, mb, mo, ep, M, N, K);
    if (e != cudaSuccess) return cuda_fail(e, "gemm2 launch");
    return MKQ_OK;
}

// Fused W4A4 GEMM + residual + LayerNorm (kLn; Gemm2Cfg<256, 8, 4, false, true>):
// one persistent CTA pair per TPC, pairs grouped np at a time; row statistics
// exchanged through `ws` (counters zeroed here, before the launch).
using LnCfg = mkq::Gemm2Cfg<256, 8, 4, false, true, 2>;      // short K (epilogue-bound): 2 boxes per warp
using LnCfgK = mkq::Gemm2Cfg<256, 8, 4, false, true, 1>;     // long K (mainloop-bound): deeper rings
using LnCfg16 = mkq::Gemm2Cfg<256, 16, 4, false, true, 1>;   // short K, 16 epilogue warps (diagnostics)
int ln_groups(int sms, int np) { return (sms / 2) / np; }
size_t ln_ws_bytes(int sms, int np) {
    const int groups = ln_groups(sms, np);
    return (size_t)groups * 2 * np * 256 * sizeof(uint64_t);
}

template <class LnCfg>
mkq_status launch_gemm2_ln_cfg(const void* a, int64_t lda, const void* w, int64_t ldw, int M, int N, int K,
                               mkq::Epi2Params& ep, void* ws, int sms, cudaStream_t st) {
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(mkq::gemm_w4a4_ln_kernel<LnCfg>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, LnCfg::kSmem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        attr_set[dev] = true;
    }
    CUtensorMap ma, mb;
    mkq_status s = make_map(&ma, a, (uint64_t)K / 2, (uint64_t)M, (uint64_t)lda, LnCfg::BK / 2, LnCfg::BM, false);
    if (s != MKQ_OK) return s;
    s = make_map(&mb, w, (uint64_t)K / 2, (uint64_t)N, (uint64_t)ldw, LnCfg::BK / 2, LnCfg::BNH, false);
    if (s != MKQ_OK) return s;
    const int np = N / 256;
    const int groups = ln_groups(sms, np);
    const int m_tiles = (M + 255) / 256;
    const int g_used = groups < m_tiles ? groups : m_tiles;
    ep.ln.flags = nullptr;
    ep.ln.stats = static_cast<float*>(ws);
    ep.ln.np = np;
    mkq::LnMaps lm;
    s = make_map_t(&lm.r, ep.ln.res, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (uint64_t)N, (uint64_t)M,
                   (uint64_t)ep.ln.ldr * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != MKQ_OK) return s;
    s = make_map_t(&lm.y, ep.ln.y, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (uint64_t)N, (uint64_t)M, (uint64_t)ep.ln.ldy * 4,
                   32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != MKQ_OK) return s;
    lm.q = lm.r;
    if (ep.ln.qbits) {
        const uint64_t qb = (uint64_t)N * ep.ln.qbits / 8;
        s = make_map_t(&lm.q, ep.ln.q, CU_TENSOR_MAP_DATA_TYPE_UINT8, qb, (uint64_t)M, (uint64_t)ep.ln.ldq,
                       (uint32_t)(32 * ep.ln.qbits / 8), 32, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (s != MKQ_OK) return s;
    }
    // the statistics slots start at tag 0 (the first use writes tag 1)
    cudaError_t e = cudaMemsetAsync(ws, 0, ln_ws_bytes(sms, np), st);
    if (e != cudaSuccess) return cuda_fail(e, "statistics reset");
    // every CTA is resident at once (one per SM, grid <= SM count): the row
    // statistics wait on other pairs of the group
    e = launch_k(mkq::gemm_w4a4_ln_kernel<LnCfg>, dim3(2 * np * g_used), dim3(LnCfg::kThreads), LnCfg::kSmem, st, 1,
                 ma, mb, ep, M, N, K, lm);
    if (e != cudaSuccess) return cuda_fail(e, "gemm_ln launch");
    return MKQ_OK;
}

int small_m_mode();   // the GEMM plan mode (below)

// ---- small-M fused GEMM + residual + LayerNorm through an N-cluster (kLnC)
using LnCCfg = mkq::GemmCfg<64, true, true>;
constexpr size_t kLnCSmem = LnCCfg::kSmem + mkq::kLnCExtra;

bool lnc_attrs() {
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return false;
    if (!done[dev]) {
        if (cudaFuncSetAttribute(mkq::gemm_lnc_kernel<LnCCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kLnCSmem) != cudaSuccess ||
            cudaFuncSetAttribute(mkq::gemm_lnc_kernel<LnCCfg>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        done[dev] = true;
    }
    return true;
}

// co-resident clusters of nt CTAs of the kLnC kernel (cached per device)
int lnc_max_clusters(int nt) {
    static int cache[64][17] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || nt < 1 || nt > 16) return 0;
    int& c = cache[dev][nt];
    if (c == 0) {
        int n = 0;
        if (lnc_attrs()) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(nt * 16));
            cfg.blockDim = dim3(LnCCfg::kThreads);
            cfg.dynamicSmemBytes = kLnCSmem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)nt;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&n, mkq::gemm_lnc_kernel<LnCCfg>, &cfg) != cudaSuccess) {
                cudaGetLastError();
                n = 0;
            }
        }
        c = n > 0 ? n : -1;
    }
    return c > 0 ? c : 0;
}

// Does the small-M N-cluster path take this W4A4 GEMM + LN?  Every cluster
// must be co-resident (one wave): ceil(M / 128) <= co-resident clusters of N/64
// CTAs (B200: one 12- or 16-CTA cluster per GPC).  MKQ_LNC=0 or the
// "never small-M" plan mode (mkq_set_small_m_mode(0), tests) disables it.
bool lnc_ok(int64_t M, int64_t N) {
    static const bool on = [] { const char* e = getenv("MKQ_LNC"); return !(e && strcmp(e, "0") == 0); }();
    if (!on || small_m_mode() == 0 || N % 64 || N / 64 < 2 || N / 64 > 16) return false;
    return (M + 127) / 128 <= lnc_max_clusters((int)(N / 64));
}

mkq_status launch_lnc(const void* a, int64_t lda, const void* w, int64_t ldw, int M, int N, int K,
                      const mkq::EpiParams& ep, const mkq::Ln2Params& ln, cudaStream_t st) {
    if (!lnc_attrs()) return fail(MKQ_ERR_CUDA, "cudaFuncSetAttribute(gemm_lnc_kernel)");
    CUtensorMap ma, mb;
    mkq_status s = make_map(&ma, a, (uint64_t)K / 2, (uint64_t)M, (uint64_t)lda, LnCCfg::BK / 2, LnCCfg::BM, true);
    if (s != MKQ_OK) return s;
    s = make_map(&mb, w, (uint64_t)K / 2, (uint64_t)N, (uint64_t)ldw, LnCCfg::BK / 2, LnCCfg::BN, true);
    if (s != MKQ_OK) return s;
    mkq::LnCParams lp;
    s = make_map_t(&lp.r, ln.res, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (uint64_t)N, (uint64_t)M, (uint64_t)ln.ldr * 4, 32,
                   32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != MKQ_OK) return s;
    s = make_out_map(&lp.y, ln.y, MKQ_OUT_F32, M, N, ln.ldy * 4);
    if (s != MKQ_OK) return s;
    lp.q = lp.y;
    if (ln.qbits) {
        s = make_out_map(&lp.q, ln.q, ln.qbits == 4 ? MKQ_OUT_I4 : MKQ_OUT_I8, M, N, ln.ldq);
        if (s != MKQ_OK) return s;
    }
    lp.g = ln.g;
    lp.b = ln.b;
    lp.eps = ln.eps;
    lp.s_q = ln.s_q;
    lp.qbits = ln.qbits;
    lp.qmin = ln.qmin;
    lp.qmax = ln.qmax;
    const int nt = N / 64, mt = (M + 127) / 128;
    cudaError_t e = launch_k(mkq::gemm_lnc_kernel<LnCCfg>, dim3((unsigned)(mt * nt)), dim3(LnCCfg::kThreads),
                             kLnCSmem, st, nt, ma, mb, lp, ep, M, N, K);
    if (e != cudaSuccess) return cuda_fail(e, "gemm_lnc launch");
    return MKQ_OK;
}

mkq_status launch_gemm2_ln(const void* a, int64_t lda, const void* w, int64_t ldw, int M, int N, int K,
                           mkq::Epi2Params& ep, void* ws, int sms, cudaStream_t st) {
    static const int boxes = [] { const char* v = getenv("MKQ_LN_BOXES"); return v ? atoi(v) : 0; }();   // diagnostics
    if (boxes == 16) return launch_gemm2_ln_cfg<LnCfg16>(a, lda, w, ldw, M, N, K, ep, ws, sms, st);
    const bool long_k = boxes ? boxes == 1 : K >= 2048;
    return long_k ? launch_gemm2_ln_cfg<LnCfgK>(a, lda, w, ldw, M, N, K, ep, ws, sms, st)
                  : launch_gemm2_ln_cfg<LnCfg>(a, lda, w, ldw, M, N, K, ep, ws, sms, st);
}

// Small-M plan (the paper's Table 2 regime of a few
// hundred to a few thousand valid tokens): when the large-tile paths would
// leave most SMs idle, the 1-CTA kernel runs 128 x 64 tiles and splits K over
// the CTAs of a thread-block cluster so that about one work unit lands on
// every SM; the partials are reduced through distributed shared memory.
// Exact: the split partials are int32 and are summed as integers (R15).
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct SmallPlan {
    bool use = false;
    int splits = 1;
    int64_t tiles = 0;
};

// -1 heuristic (default), 0 never, 1 always: mkq_set_small_m_mode() or the
// MKQ_SMALL_M environment variable (tests and diagnostics).
std::atomic<int> g_small_mode{[] { const char* e = getenv("MKQ_SMALL_M"); return e ? atoi(e) : -1; }()};

// cudaOccupancyMaxActiveClusters of the small-M kernel per cluster size
// (cached per device; int4 and int8 variants use the same shared memory
// class, one CTA per SM).
int max_clusters(int csize) {
    static int cache[64][9] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || csize < 1 || csize > 8) return 0;
    int& c = cache[dev][csize];
    if (c == 0) {
        using Cfg = mkq::GemmCfg<64, true, true>;
        cudaFuncSetAttribute(mkq::gemm_i8tc_kernel<Cfg, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(csize * 64));
        cfg.blockDim = dim3(Cfg::kThreads);
        cfg.dynamicSmemBytes = Cfg::kSmem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)csize;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, mkq::gemm_i8tc_kernel<Cfg, true>, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            n = 1;
        }
        c = n;
    }
    return c;
}

int small_m_mode() { return g_small_mode.load(std::memory_order_relaxed); }

// Single wave only: 128 x 64 tiles if they fit one per SM, else the
// large-tile paths.  K is split over a cluster while the clusters
// still fit (one wave, <= 4 CTAs per cluster, >= 2 K-blocks per split).
SmallPlan plan_small(int64_t M, int64_t N, int64_t K, int sms, bool int4) {
    SmallPlan p;
    const int mode = small_m_mode();
    if (mode == 0) return p;
    const int64_t mt = (M + 127) / 128;
    const int64_t t64 = mt * ((N + 63) / 64);
    // (128 x 128 tiles measured slower than the 2-CTA 256 x 256 path at
    // Table-2 sizes: t64 > sms goes to the large-tile paths)
    if (t64 <= sms || mode == 1) {
        p.tiles = t64;
    } else {
        return p;
    }
    p.use = true;
    const int64_t nk = (K + 127) / 128;
    int64_t sp = sms / std::max<int64_t>(p.tiles, 1);
    // K split only for long K: the cluster reduction (barrier + DSMEM round
    // trip + a second store pass) costs more than it saves below 12 x 128 K
    // per split for int4 (256-K stages), and always for int8 at Table-2 sizes
    // (440 tokens: O 7.2 -> 5.3 us int4 / 6.5 -> 4.5 us int8 unsplit; FFN2
    // int4 9.3 us split 2 vs 9.9 unsplit, int8 8.3 vs 7.9)
    static const int min_kb = [] { const char* e = getenv("MKQ_SPLIT_MIN_KB"); return e ? atoi(e) : 12; }();
    sp = int4 ? std::min<int64_t>(sp, nk / std::max(min_kb, 1)) : 1;
    static const int max_split = [] { const char* e = getenv("MKQ_MAX_SPLIT"); return e ? atoi(e) : 4; }();
    sp = std::min<int64_t>(sp, max_split);   // clusters of <= 4 full-SM CTAs co-reside in a GPC
    p.splits = (int)std::max<int64_t>(sp, 1);
    // every cluster must be co-resident (one wave)
    while (p.splits > 1 && p.tiles > max_clusters(p.splits)) --p.splits;
    return p;
}

mkq_status gemm_common(bool int4, const void* a, int64_t lda, const void* w, int64_t ldw, int64_t M, int64_t N,
                       int64_t K, float s_a, const float* s_w, const float* bias, const mkq_epilogue* epi, void* out,
                       int64_t ldo, void* ws, size_t ws_bytes, void* stream) {
    (void)ws;
    (void)ws_bytes;
    mkq_epilogue e{MKQ_OUT_F32, 0, 1.0f, 0, 0, nullptr};
    if (epi) e = *epi;
    if (M < 0 || N < 0 || K < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (M == 0) return MKQ_OK;
    if (!a || !w || !s_w || !out) return fail(MKQ_ERR_NULL, "a, w, s_w and out are required");
    if (N == 0 || N % 32) return fail(MKQ_ERR_SHAPE, "N=%lld must be a positive multiple of 32", (long long)N);
    if (K < 32 || K % 32 || K > MKQ_MAX_K)
        return fail(MKQ_ERR_SHAPE, "K=%lld must be a multiple of 32 in [32, %d]", (long long)K, MKQ_MAX_K);
    if (M > (1ll << 31) - 256 || N > (1 << 24)) return fail(MKQ_ERR_SHAPE, "M or N too large");
    const int64_t krow = int4 ? K / 2 : K;
    int64_t orow;
    switch (e.out) {
    case MKQ_OUT_F32: case MKQ_OUT_I32: orow = 4 * N; break;
    case MKQ_OUT_BF16: case MKQ_OUT_F16: orow = 2 * N; break;
    case MKQ_OUT_I8: orow = N; break;
    case MKQ_OUT_I4: orow = N / 2; break;
    default: return fail(MKQ_ERR_RANGE, "unknown epilogue mode %d", e.out);
    }
    if (lda < krow || ldw < krow || ldo < orow) return fail(MKQ_ERR_SHAPE, "leading dimension smaller than a row");
    if (!aligned16(a) || !aligned16(w) || !aligned16(out) || lda % 16 || ldw % 16 || ldo % 16)
        return fail(MKQ_ERR_ALIGN, "pointers and leading dimensions must be 16-byte aligned");
    if (!finite_pos(s_a)) return fail(MKQ_ERR_SCALE, "s_a must be > 0 and finite");
    const bool requant = e.out == MKQ_OUT_I4 || e.out == MKQ_OUT_I8;
    if (requant) {
        if (!finite_pos(e.s_out)) return fail(MKQ_ERR_SCALE, "s_out must be > 0 and finite");
        if (!code_range_ok(e.out == MKQ_OUT_I4 ? 4 : 8, e.qmin_out, e.qmax_out))
            return fail(MKQ_ERR_RANGE, "qmin_out/qmax_out not representable");
    }
    if (e.gelu != 0 && e.gelu != 1) return fail(MKQ_ERR_RANGE, "gelu must be 0 or 1");
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;

    PdlScope pdl_scope(M);
    mkq::EpiParams ep;
    ep.mode = e.out;
    ep.gelu = e.out == MKQ_OUT_I32 ? 0 : e.gelu;
    ep.s_a = s_a;
    ep.s_w = s_w;
    ep.bias = bias;
    ep.s_out = e.s_out;
    ep.qmin = e.qmin_out;
    ep.qmax = e.qmax_out;
    ep.out = out;
    ep.ldo_bytes = ldo;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // mma.sync small-M kernel: latency-first (mode 2 forces it; heuristic:
    // set by MKQ_MMA_SMALL_M rows, default 0 = off until measured)
    static const int mma_rows = [] { const char* e = getenv("MKQ_MMA_SMALL_M"); return e ? atoi(e) : 0; }();
    if (small_m_mode() == 2 || (small_m_mode() == -1 && M <= mma_rows)) {
        PdlScope pdl_scope_m(M);
        static bool attr[2][64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        const int ii = int4 ? 1 : 0;
        if (!attr[ii][dev]) {
            cudaError_t e = int4 ? cudaFuncSetAttribute(mkq::gsm::gemm_mma_small_kernel<true>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        mkq::gsm::Cfg<true>::kSmem)
                                 : cudaFuncSetAttribute(mkq::gsm::gemm_mma_small_kernel<false>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        mkq::gsm::Cfg<false>::kSmem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(gemm_mma_small)");
            attr[ii][dev] = true;
        }
        const dim3 grid((unsigned)((N + mkq::gsm::BN - 1) / mkq::gsm::BN), (unsigned)((M + mkq::gsm::BM - 1) / mkq::gsm::BM));
        cudaError_t e = int4 ? launch_k(mkq::gsm::gemm_mma_small_kernel<true>, grid, dim3(mkq::gsm::kThreads),
                                        mkq::gsm::Cfg<true>::kSmem, st, 1, static_cast<const uint8_t*>(a), lda,
                                        static_cast<const uint8_t*>(w), ldw, ep, (int)M, (int)N, (int)K)
                             : launch_k(mkq::gsm::gemm_mma_small_kernel<false>, grid, dim3(mkq::gsm::kThreads),
                                        mkq::gsm::Cfg<false>::kSmem, st, 1, static_cast<const uint8_t*>(a), lda,
                                        static_cast<const uint8_t*>(w), ldw, ep, (int)M, (int)N, (int)K);
        if (e != cudaSuccess) return cuda_fail(e, "gemm_mma_small launch");
        return MKQ_OK;
    }
    const SmallPlan sp = plan_small(M, N, K, sms, int4);
    if (sp.use) {
        if (int4) return launch_gemm<mkq::GemmCfg<64, true, true>, true>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st, sp.splits);
        return launch_gemm<mkq::GemmCfg<64, false>, true>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st, sp.splits);
    }
    // int4 small M with more 128 x 64 tiles than SMs (Table-2 QKV at 537-681 tokens):
    // 128 x 128 tiles of the same A-in-TMEM plan, unsplit, when they fit one wave
    // (plain outputs; the FFN1 requant keeps the compact-table CTA-pair path)
    if (int4 && small_m_mode() != 0 && N % 128 == 0 && e.out != MKQ_OUT_I4 && e.out != MKQ_OUT_I8 &&
        ((M + 127) / 128) * (N / 128) <= sms && ((M + 127) / 128) * ((N + 63) / 64) > sms)
        return launch_gemm<mkq::GemmCfg<128, true, true>, true>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st, 1);
    const bool wide = (N % 256 == 0) && (M > 128 * sms / 2 || (M / 128 + 1) * (N / 256) >= sms);
    static const int path_override = [] {   // MKQ_GEMM_PATH=1cta|2cta (diagnostics)
        const char* v = getenv("MKQ_GEMM_PATH");
        return v ? (strcmp(v, "1cta") == 0 ? 1 : (strcmp(v, "2cta") == 0 ? 2 : 0)) : 0;
    }();
    const bool two_cta = path_override == 2 ? (N % 128 == 0) : (path_override == 1 ? false : (M > 128 && N % 128 == 0));
    if (int4 && two_cta) {
        mkq::Epi2Params p2{ep, (e.out == MKQ_OUT_I4 || e.out == MKQ_OUT_I8) ? e.requant_table : nullptr};
        if (p2.table && !aligned16(p2.table)) return fail(MKQ_ERR_ALIGN, "requant_table must be 16-byte aligned");
        // K <= 1024 tiles are epilogue-bound (8 K-blocks per tile): 16 epilogue + 4
        // unpack warps; longer K keeps 8 + 8 (mainloop-bound)
        static const int epi_override = [] { const char* v = getenv("MKQ_EPI_WARPS"); return v ? atoi(v) : 0; }();
        const bool many_epi = epi_override ? epi_override == 16 : K <= 1024;
        static const bool no_lut4 = getenv("MKQ_NO_LUT4") != nullptr;   // diagnostics
        if (N % 256 == 0) {
            // (8 unpack warps with 88-register epilogue warps measured 7% slower)
            static const int lut4_epi = [] { const char* v = getenv("MKQ_LUT4_EPI"); return v ? atoi(v) : 16; }();
            if (many_epi && e.out == MKQ_OUT_I4 && p2.table && !no_lut4) {
                // small M (paper Table 2: FFN1 at 440-681 tokens): 256 x 128 pair
                // tiles put twice as many SMs on the GEMM as 256 x 256 ones
                static const int lut128_pairs = [] { const char* v = getenv("MKQ_LUT128_PAIRS"); return v ? atoi(v) : -1; }();
                const int64_t pairs256 = ((M + 255) / 256) * (N / 256);
                if (pairs256 * 4 <= sms && (lut128_pairs < 0 || pairs256 <= lut128_pairs))
                    return launch_gemm2<mkq::Gemm2Cfg<128, 8, 4, true>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
                if (lut4_epi == 8)
                    return launch_gemm2<mkq::Gemm2Cfg<256, 8, 4, true>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
                if (lut4_epi == 168)
                    return launch_gemm2<mkq::Gemm2Cfg<256, 16, 8, true>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
                return launch_gemm2<mkq::Gemm2Cfg<256, 16, 4, true>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
            }
            if (many_epi)
                return launch_gemm2<mkq::Gemm2Cfg<256, 16, 4>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
            return launch_gemm2<mkq::Gemm2Cfg<256>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
        }
        return launch_gemm2<mkq::Gemm2Cfg<128>>(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, sms, st);
    }
    if (int4) {
        if (wide) return launch_gemm<mkq::GemmCfg<256, true>>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st);
        return launch_gemm<mkq::GemmCfg<128, true>>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st);
    }
    if (wide) return launch_gemm<mkq::GemmCfg<256, false>>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st);
    return launch_gemm<mkq::GemmCfg<128, false>>(a, lda, w, ldw, (int)M, (int)N, (int)K, ep, sms, st);
}

int grid_for(int64_t work, int threads, int sms) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)sms * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}


// Launch the quantize/pack kernels; the scale is a device pointer (scale_dev)
// or, when that is NULL, the per-tensor value s_val.  Arguments validated.
mkq_status quantize_internal(const float* x, int64_t rows, int64_t cols, int64_t ldx, const float* scale_dev,
                             float s_val, int per_row, int bits, int qmin, int qmax, void* q, int64_t ldq, int sms,
                             cudaStream_t st) {
    PdlScope pdl_scope(rows);
    const bool vec = cols % 8 == 0 && ldx % 4 == 0 && aligned16(x) &&
                     (bits == 4 ? (ldq % 4 == 0 && (reinterpret_cast<uintptr_t>(q) & 3) == 0)
                                : (ldq % 8 == 0 && (reinterpret_cast<uintptr_t>(q) & 7) == 0));
    uint8_t* qq = static_cast<uint8_t*>(q);
    if (vec) {
        const int g = grid_for(rows * (cols / 8), 256, sms);
        if (bits == 4) {
            if (per_row) launch_k(mkq::quantize_pack_vec_kernel<4, true>, dim3(g), dim3(256), 0, st, 1, x, rows, cols, ldx, scale_dev, s_val, qmin, qmax, qq, ldq);
            else launch_k(mkq::quantize_pack_vec_kernel<4, false>, dim3(g), dim3(256), 0, st, 1, x, rows, cols, ldx, scale_dev, s_val, qmin, qmax, qq, ldq);
        } else {
            if (per_row) launch_k(mkq::quantize_pack_vec_kernel<8, true>, dim3(g), dim3(256), 0, st, 1, x, rows, cols, ldx, scale_dev, s_val, qmin, qmax, qq, ldq);
            else launch_k(mkq::quantize_pack_vec_kernel<8, false>, dim3(g), dim3(256), 0, st, 1, x, rows, cols, ldx, scale_dev, s_val, qmin, qmax, qq, ldq);
        }
    } else {
        const int g = grid_for(rows * (bits == 4 ? cols / 2 : cols), 256, sms);
        if (bits == 4) launch_k(mkq::quantize_pack_any_kernel<4>, dim3(g), dim3(256), 0, st, 1, x, rows, cols, ldx, scale_dev, s_val, per_row, qmin, qmax, qq, ldq);
        else launch_k(mkq::quantize_pack_any_kernel<8>, dim3(g), dim3(256), 0, st, 1, x, rows, cols, ldx, scale_dev, s_val, per_row, qmin, qmax, qq, ldq);
    }
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "quantize launch");
}

}  // namespace

extern "C" {

const char* mkq_status_string(int s) {
    switch (s) {
    case MKQ_OK: return "MKQ_OK";
    case MKQ_ERR_NULL: return "MKQ_ERR_NULL";
    case MKQ_ERR_SHAPE: return "MKQ_ERR_SHAPE";
    case MKQ_ERR_ALIGN: return "MKQ_ERR_ALIGN";
    case MKQ_ERR_SCALE: return "MKQ_ERR_SCALE";
    case MKQ_ERR_RANGE: return "MKQ_ERR_RANGE";
    case MKQ_ERR_DEVICE: return "MKQ_ERR_DEVICE";
    case MKQ_ERR_WORKSPACE: return "MKQ_ERR_WORKSPACE";
    case MKQ_ERR_CUDA: return "MKQ_ERR_CUDA";
    default: return "MKQ_ERR_UNKNOWN";
    }
}

const char* mkq_last_error(void) { return g_err; }

int mkq_version(void) { return MKQ_VERSION; }

mkq_status mkq_quantize_pack(const float* x, int64_t rows, int64_t cols, int64_t ldx, const float* scale,
                             int per_row, int bits, int qmin, int qmax, void* q, int64_t ldq, void* stream) {
    if (rows < 0 || cols < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (rows == 0 || cols == 0) return MKQ_OK;
    if (!x || !scale || !q) return fail(MKQ_ERR_NULL, "x, scale and q are required");
    if (bits != 4 && bits != 8) return fail(MKQ_ERR_RANGE, "bits must be 4 or 8");
    if (bits == 4 && cols % 2) return fail(MKQ_ERR_SHAPE, "int4 needs an even column count");
    if (ldx < cols || ldq < (bits == 4 ? cols / 2 : cols)) return fail(MKQ_ERR_SHAPE, "leading dimension too small");
    if (per_row != 0 && per_row != 1) return fail(MKQ_ERR_RANGE, "per_row must be 0 or 1");
    if (!code_range_ok(bits, qmin, qmax)) return fail(MKQ_ERR_RANGE, "qmin/qmax not representable in %d bits", bits);
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    return quantize_internal(x, rows, cols, ldx, scale, 0.0f, per_row, bits, qmin, qmax, q, ldq, sms,
                             static_cast<cudaStream_t>(stream));
}

mkq_status mkq_absmax_scale(const float* x, int64_t rows, int64_t cols, int64_t ldx, int per_row, float l_max,
                            float* s_out, void* stream) {
    if (rows < 0 || cols < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (!x || !s_out) return fail(MKQ_ERR_NULL, "x and s_out are required");
    if (rows == 0 || cols == 0) return fail(MKQ_ERR_SHAPE, "empty input has no scale");
    if (ldx < cols) return fail(MKQ_ERR_SHAPE, "leading dimension too small");
    if (!finite_pos(l_max)) return fail(MKQ_ERR_SCALE, "l_max must be > 0 and finite");
    if (per_row != 0 && per_row != 1) return fail(MKQ_ERR_RANGE, "per_row must be 0 or 1");
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int vec = (cols % 4 == 0 && ldx % 4 == 0 && aligned16(x)) ? 1 : 0;
    const int g = grid_for(rows * 32, 256, sms);
    if (per_row) {
        mkq::absmax_rows_kernel<<<g, 256, 0, st>>>(x, rows, cols, ldx, vec, l_max, s_out, nullptr);
    } else {
        cudaMemsetAsync(s_out, 0, sizeof(float), st);
        unsigned int* bitsp = reinterpret_cast<unsigned int*>(s_out);
        mkq::absmax_rows_kernel<<<g, 256, 0, st>>>(x, rows, cols, ldx, vec, l_max, nullptr, bitsp);
        mkq::absmax_finalize_kernel<<<1, 1, 0, st>>>(bitsp, l_max, s_out);
    }
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "absmax launch");
}

mkq_status mkq_gemm_w4a4(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t M, int64_t N, int64_t K,
                         float s_a, const float* s_w, const float* bias, const mkq_epilogue* epi, void* out,
                         int64_t ldo, void* ws, size_t ws_bytes, void* stream) {
    return gemm_common(true, a, lda, w, ldw, M, N, K, s_a, s_w, bias, epi, out, ldo, ws, ws_bytes, stream);
}

mkq_status mkq_gemm_w8a8(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t M, int64_t N, int64_t K,
                         float s_a, const float* s_w, const float* bias, const mkq_epilogue* epi, void* out,
                         int64_t ldo, void* ws, size_t ws_bytes, void* stream) {
    return gemm_common(false, a, lda, w, ldw, M, N, K, s_a, s_w, bias, epi, out, ldo, ws, ws_bytes, stream);
}

void mkq_set_small_m_mode(int mode) { g_small_mode.store(mode < 0 ? -1 : (mode > 2 ? 2 : mode)); }

// ------------------------------------------------------------------ NEXT(4) fused all-gather
using GatherCfg = mkq::Gemm2Cfg<256, 16, 4, true>;

static int gather_grid(int64_t M, int64_t N, int sms) {
    const int64_t tiles = ((M + 2 * GatherCfg::BM - 1) / (2 * GatherCfg::BM)) * ((N + GatherCfg::BN - 1) / GatherCfg::BN);
    const int clusters = (int)(tiles < sms / 2 ? tiles : sms / 2);
    return 2 * clusters;
}

int mkq_gemm_gather_arrivals(int64_t M, int64_t N) {
    int sms = 148;
    if (check_device(&sms) != MKQ_OK) sms = 148;
    return M > 0 && N > 0 ? gather_grid(M, N, sms) : 0;
}

mkq_status mkq_gemm_w4a4_gather(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t M, int64_t N,
                                int64_t K, float s_a, const float* s_w, const float* bias, const mkq_epilogue* epi,
                                void* const* outs, int nout, int64_t col0, int64_t ldo, uint32_t* const* counters,
                                void* stream) {
    if (M < 0 || N < 0 || K < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (M == 0) return MKQ_OK;
    if (!a || !w || !s_w || !epi || !outs || !counters) return fail(MKQ_ERR_NULL, "a, w, s_w, epi, outs, counters");
    if (nout < 1 || nout > mkq::kMaxGather) return fail(MKQ_ERR_RANGE, "nout must be in [1, %d]", mkq::kMaxGather);
    if (epi->out != MKQ_OUT_I4 || !epi->requant_table) return fail(MKQ_ERR_RANGE, "the fused all-gather is the int4 requant (table) epilogue");
    if (!code_range_ok(4, epi->qmin_out, epi->qmax_out)) return fail(MKQ_ERR_RANGE, "qmin/qmax");
    if (!finite_pos(epi->s_out) || !finite_pos(s_a)) return fail(MKQ_ERR_SCALE, "s_a and s_out must be > 0 and finite");
    if (N % 256 || K % 32 || K > 1024 || K < 32) return fail(MKQ_ERR_SHAPE, "N % 256 == 0 and K in [32, 1024], K % 32 == 0");
    if (col0 < 0 || col0 % 32 || ldo < (col0 + N) / 2 || ldo % 16) return fail(MKQ_ERR_SHAPE, "col0 / ldo");
    if (lda < K / 2 || ldw < K / 2 || lda % 16 || ldw % 16 || !aligned16(a) || !aligned16(w) || !aligned16(epi->requant_table))
        return fail(MKQ_ERR_ALIGN, "operands");
    for (int g = 0; g < nout; ++g) {
        if (!outs[g] || !counters[g]) return fail(MKQ_ERR_NULL, "outs[%d] / counters[%d]", g, g);
        if (!aligned16(outs[g]) || (reinterpret_cast<uintptr_t>(counters[g]) & 3)) return fail(MKQ_ERR_ALIGN, "outs / counters");
    }
    int sms = 0;
    mkq_status st = check_device(&sms);
    if (st != MKQ_OK) return st;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(mkq::gemm_w4a4_gather_kernel<GatherCfg>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, GatherCfg::kSmem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        attr_set[dev] = true;
    }
    mkq::EpiParams ep{MKQ_OUT_I4, epi->gelu, s_a, s_w, bias, epi->s_out, epi->qmin_out, epi->qmax_out, outs[0], ldo};
    mkq::Epi2Params p2{ep, epi->requant_table, {}};
    CUtensorMap ma, mb;
    st = make_map(&ma, a, (uint64_t)K / 2, (uint64_t)M, (uint64_t)lda, GatherCfg::BK / 2, GatherCfg::BM, false);
    if (st != MKQ_OK) return st;
    st = make_map(&mb, w, (uint64_t)K / 2, (uint64_t)N, (uint64_t)ldw, GatherCfg::BK / 2, GatherCfg::BNH, false);
    if (st != MKQ_OK) return st;
    mkq::GatherMaps gm{};
    for (int g = 0; g < nout; ++g) {
        // the gathered buffer is [M, >= col0 + N] codes; its row stride ldo bytes
        st = make_out_map(&gm.m[g], outs[g], MKQ_OUT_I4, M, 2 * ldo, ldo);
        if (st != MKQ_OK) return st;
        gm.counters[g] = counters[g];
    }
    gm.n = nout;
    gm.col0 = (int)col0;
    PdlScope pdl_scope(M);
    cudaError_t e = launch_k(mkq::gemm_w4a4_gather_kernel<GatherCfg>, dim3(gather_grid(M, N, sms)),
                             dim3(GatherCfg::kThreads), GatherCfg::kSmem, static_cast<cudaStream_t>(stream), 1, ma, mb,
                             p2, (int)M, (int)N, (int)K, gm);
    if (e != cudaSuccess) return cuda_fail(e, "gemm_gather launch");
    return MKQ_OK;
}

mkq_status mkq_wait_counter(const uint32_t* counter, uint32_t target, void* stream) {
    if (!counter) return fail(MKQ_ERR_NULL, "counter");
    mkq::wait_counter_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(counter, target);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "wait_counter launch");
}

typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

mkq_status mkq_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset) {
    if (!dev_ptr || !handle || !offset) return fail(MKQ_ERR_NULL, "dev_ptr / handle / offset");
    static AddrRangeFn range = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
                       q == cudaDriverEntryPointSuccess
                   ? reinterpret_cast<AddrRangeFn>(p)
                   : nullptr;
    }();
    if (!range) return fail(MKQ_ERR_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr));
    if (r != CUDA_SUCCESS) return fail(MKQ_ERR_CUDA, "cuMemGetAddressRange failed (%d)", (int)r);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    return MKQ_OK;
}

mkq_status mkq_ipc_open_handle(const void* handle, void** dev_ptr) {
    if (!dev_ptr || !handle) return fail(MKQ_ERR_NULL, "dev_ptr / handle");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

mkq_status mkq_ipc_close(void* dev_ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

size_t mkq_gemm_workspace_size(int64_t, int64_t, int64_t) { return 0; }

size_t mkq_gemm_residual_ln_workspace_size(int64_t M, int64_t N) {
    if (M <= 0 || N <= 0 || N % 256) return 0;
    int sms = 148;
    if (check_device(&sms) != MKQ_OK) sms = 148;
    return ln_ws_bytes(sms, (int)(N / 256));
}

mkq_status mkq_gemm_residual_ln(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t M, int64_t N,
                                int64_t K, float s_a, const float* s_w, const float* bias, const float* res,
                                int64_t ldr, const float* gamma, const float* beta, float eps, float* y, int64_t ldy,
                                int q_bits, float s_q, int qmin, int qmax, void* q, int64_t ldq, void* ws,
                                size_t ws_bytes, void* stream) {
    if (M < 0 || N < 0 || K < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (M == 0) return MKQ_OK;
    if (!a || !w || !s_w || !res || !gamma || !beta || !y || !ws) return fail(MKQ_ERR_NULL, "a, w, s_w, res, gamma, beta, y and ws are required");
    if (q_bits && !q) return fail(MKQ_ERR_NULL, "q is required when q_bits != 0");
    if (N % 256 || N < 256 || N > 1024) return fail(MKQ_ERR_SHAPE, "N must be 256, 512, 768 or 1024");
    if (K <= 0 || K % 32 || K > MKQ_MAX_K) return fail(MKQ_ERR_SHAPE, "K must be a positive multiple of 32 <= %d", MKQ_MAX_K);
    if (lda < K / 2 || ldw < K / 2 || lda % 16 || ldw % 16) return fail(MKQ_ERR_ALIGN, "lda/ldw: >= K/2 bytes, multiples of 16");
    if (ldr < N || ldy < N || ldr % 4 || ldy % 4) return fail(MKQ_ERR_SHAPE, "ldr/ldy must be >= N and multiples of 4");
    if (!aligned16(a) || !aligned16(w) || !aligned16(res) || !aligned16(y) || !aligned16(ws))
        return fail(MKQ_ERR_ALIGN, "a, w, res, y and ws must be 16-byte aligned");
    if (!finite_pos(s_a)) return fail(MKQ_ERR_SCALE, "s_a must be > 0 and finite");
    if (!(eps >= 0.0f) || !std::isfinite(eps)) return fail(MKQ_ERR_SCALE, "eps must be finite and >= 0");
    if (q_bits) {
        if (q_bits != 4 && q_bits != 8) return fail(MKQ_ERR_RANGE, "q_bits must be 0, 4 or 8");
        if (!finite_pos(s_q)) return fail(MKQ_ERR_SCALE, "s_q must be > 0 and finite");
        if (!code_range_ok(q_bits, qmin, qmax)) return fail(MKQ_ERR_RANGE, "qmin/qmax");
        if (ldq < (q_bits == 4 ? N / 2 : N) || ldq % 16 || !aligned16(q)) return fail(MKQ_ERR_ALIGN, "q rows: 16-byte aligned, ldq >= N*q_bits/8");
    }
    int sms = 0;
    mkq_status st = check_device(&sms);
    if (st != MKQ_OK) return st;
    if (ws_bytes < ln_ws_bytes(sms, (int)(N / 256))) return fail(MKQ_ERR_WORKSPACE, "workspace too small");
    mkq::Epi2Params p2{};
    p2.e = mkq::EpiParams{mkq::OUT_F32, 0, s_a, s_w, bias, 1.0f, 0, 0, y, ldy * 4};
    p2.table = nullptr;
    p2.ln = mkq::Ln2Params{res, ldr, gamma, beta, eps, y, ldy, static_cast<uint8_t*>(q), ldq, q_bits, qmin, qmax,
                           s_q, nullptr, nullptr, (int)(N / 256)};
    PdlScope pdl_scope(M);
    if (lnc_ok(M, N)) return launch_lnc(a, lda, w, ldw, (int)M, (int)N, (int)K, p2.e, p2.ln, static_cast<cudaStream_t>(stream));
    return launch_gemm2_ln(a, lda, w, ldw, (int)M, (int)N, (int)K, p2, ws, sms, static_cast<cudaStream_t>(stream));
}

size_t mkq_requant_table_size(void) { return mkq::rq::kTableBytes; }

}  // extern "C"

namespace mkq {
namespace rq {
__global__ void init_kernel(Header* h, float y_lo, float y_hi, float inv_w, float y_zero, int ncell, int code_lo,
                            int code_hi, int gelu, int qmin, int qmax, float s) {
    Header v{};
    v.y_lo = y_lo; v.y_hi = y_hi; v.inv_w = inv_w; v.y_zero = y_zero;
    v.c0 = __fmul_rn(-y_lo, inv_w);
    v.ncell = ncell; v.code_lo = code_lo; v.code_hi = code_hi; v.valid = 0;
    v.gelu = gelu; v.qmin = qmin; v.qmax = qmax; v.nchg = 0; v.s_out = s;
    *h = v;
}
}  // namespace rq
}  // namespace mkq

extern "C" {

mkq_status mkq_requant_table(int gelu, float s_out, int qmin, int qmax, void* table, size_t table_bytes,
                             void* stream) {
    if (!table) return fail(MKQ_ERR_NULL, "table is required");
    if (table_bytes < mkq::rq::kTableBytes) return fail(MKQ_ERR_WORKSPACE, "table needs %zu bytes", mkq::rq::kTableBytes);
    if (!aligned16(table)) return fail(MKQ_ERR_ALIGN, "table must be 16-byte aligned");
    if (!finite_pos(s_out) || s_out > 1e30f || s_out < 1e-30f) return fail(MKQ_ERR_SCALE, "s_out out of range");
    if (gelu != 0 && gelu != 1) return fail(MKQ_ERR_RANGE, "gelu must be 0 or 1");
    const int bits = (qmin >= -8 && qmax <= 7) ? 4 : 8;
    if (!code_range_ok(bits, qmin, qmax) || qmin > 0 || qmax < 0) return fail(MKQ_ERR_RANGE, "need qmin <= 0 <= qmax");
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    using namespace mkq::rq;
    float y_lo, y_hi;
    int code_lo, code_hi = qmax;
    if (gelu) {
        y_lo = -5.6f;
        y_hi = fmaxf(5.6f, (float)(qmax + 1) * s_out);
        code_lo = 0;
    } else {
        y_lo = (float)(qmin - 1) * s_out;
        y_hi = (float)(qmax + 1) * s_out;
        code_lo = qmin;
    }
    const float y_zero = 0.49f * s_out;
    if (!(y_lo < -y_zero && y_zero < y_hi)) return fail(MKQ_ERR_SCALE, "s_out too large for the table range");
    const float inv_w = (float)kCells / (y_hi - y_lo);
    uint32_t bz, bh, bl;
    memcpy(&bz, &y_zero, 4);
    memcpy(&bh, &y_hi, 4);
    const float ny_lo = -y_lo;
    memcpy(&bl, &ny_lo, 4);
    const uint32_t np = bh - bz + 1, nn = bl - bz + 1;
    Header* h = static_cast<Header*>(table);
    uint2* cells = reinterpret_cast<uint2*>(h + 1);
    Header4* h4 = reinterpret_cast<Header4*>(static_cast<uint8_t*>(table) + kOff4);
    uint32_t* cells4 = reinterpret_cast<uint32_t*>(h4 + 1);
    Change* chg = reinterpret_cast<Change*>(reinterpret_cast<uint8_t*>(cells4) + kCells4 * 4);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    init_kernel<<<1, 1, 0, st>>>(h, y_lo, y_hi, inv_w, y_zero, kCells, code_lo, code_hi, gelu, qmin, qmax, s_out);
    scan_kernel<<<sms * 8, 256, 0, st>>>(h, chg, bz, np, bz, nn);
    finalize_kernel<<<1, 32, 0, st>>>(h, cells, chg);
    verify_kernel<<<sms * 8, 256, 0, st>>>(h, cells, bz, np, bz, nn);
    finalize4_kernel<<<1, 32, 0, st>>>(h, h4, cells4, chg);
    verify4_kernel<<<sms * 8, 256, 0, st>>>(h, h4, cells4, bz, np, bz, nn);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "requant table launch");
}

mkq_status mkq_attention(const void* qkv, int64_t ld, int64_t batch, int64_t max_seq, const int32_t* cu,
                         int64_t tokens, int heads, int head_dim, int out_mode, float s_out, int qmin, int qmax,
                         void* out, int64_t ldo, void* stream) {
    if (batch < 0 || max_seq < 0 || tokens < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (batch == 0 || tokens == 0) return MKQ_OK;
    if (!qkv || !out) return fail(MKQ_ERR_NULL, "qkv and out are required");
    if (head_dim != 64) return fail(MKQ_ERR_SHAPE, "head_dim must be 64");
    if (heads <= 0 || heads > 65535) return fail(MKQ_ERR_SHAPE, "heads out of range");
    if (max_seq <= 0 || max_seq > 1024) return fail(MKQ_ERR_SHAPE, "max_seq must be in [1, 1024]");
    if (batch > 65535) return fail(MKQ_ERR_SHAPE, "batch must be <= 65535");
    if (!cu && tokens != batch * max_seq) return fail(MKQ_ERR_SHAPE, "tokens != batch*max_seq without cu_seqlens");
    const int64_t hidden = (int64_t)heads * 64;
    if (ld < 3 * hidden) return fail(MKQ_ERR_SHAPE, "ld_qkv smaller than 3*hidden");
    if (!aligned16(qkv) || ld % 8) return fail(MKQ_ERR_ALIGN, "qkv rows must be 16-byte aligned");
    int64_t orow;
    if (out_mode == MKQ_OUT_F32) orow = 4 * hidden;
    else if (out_mode == MKQ_OUT_I4) orow = hidden / 2;
    else if (out_mode == MKQ_OUT_I8) orow = hidden;
    else return fail(MKQ_ERR_RANGE, "attention out_mode must be F32, I4 or I8");
    if (ldo < orow) return fail(MKQ_ERR_SHAPE, "ldo smaller than a row");
    if (!aligned16(out) || ldo % 16) return fail(MKQ_ERR_ALIGN, "out rows must be 16-byte aligned");
    if (out_mode != MKQ_OUT_F32) {
        if (!finite_pos(s_out)) return fail(MKQ_ERR_SCALE, "s_out must be > 0 and finite");
        if (!code_range_ok(out_mode == MKQ_OUT_I4 ? 4 : 8, qmin, qmax)) return fail(MKQ_ERR_RANGE, "qmin/qmax");
    }
    mkq_status s = check_device();
    if (s != MKQ_OK) return s;
    static const int attn_env = [] {   // MKQ_ATTN=mma|pp forces a kernel (diagnostics)
        const char* v = getenv("MKQ_ATTN");
        if (v && strcmp(v, "mma") == 0) return 1;
        if (v && strcmp(v, "pp") == 0) return 2;
        return -1;
    }();
    // Short sequences (max_seq <= 128: BERT-base configs, the paper's Table 2
    // batches of ~30 valid tokens per sequence): the mma.sync flash kernel,
    // 64-query CTAs that exit early past the sequence end, beats the
    // persistent tcgen05 kernel's 2 x 128-query tiles (6.6 vs 11.2 us at 440
    // valid tokens, 12.7 vs 28.7 us at 2298); long sequences: tcgen05.
    const int attn_path = attn_env >= 0 ? attn_env : (max_seq <= 128 ? 1 : 2);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PdlScope pdl_scope(tokens);
    if (attn_path == 2) {
        const int mi = out_mode == MKQ_OUT_F32 ? 0 : (out_mode == MKQ_OUT_I4 ? 1 : 2);
        auto kern = mi == 0 ? mkq::attnpp::attn_pp_kernel<0>
                            : (mi == 1 ? mkq::attnpp::attn_pp_kernel<3> : mkq::attnpp::attn_pp_kernel<4>);
        static bool attr_set[3][64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!attr_set[mi][dev]) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, mkq::attnpp::kSmem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(attn_pp)");
            attr_set[mi][dev] = true;
        }
        CUtensorMap mq, mkv;
        s = make_map_t(&mq, qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)(3 * hidden), (uint64_t)tokens,
                       (uint64_t)ld * 2, 64, mkq::attnpp::kBQ, CU_TENSOR_MAP_SWIZZLE_128B);
        if (s != MKQ_OK) return s;
        s = make_map_t(&mkv, qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)(3 * hidden), (uint64_t)tokens,
                       (uint64_t)ld * 2, 64, mkq::attnpp::kBK, CU_TENSOR_MAP_SWIZZLE_128B);
        if (s != MKQ_OK) return s;
        mkq::attn2::Params p;
        p.cu = cu;
        p.seq = (int)max_seq;
        p.hidden = (int)hidden;
        p.out_mode = out_mode;
        p.s_out = s_out;
        p.qmin = qmin;
        p.qmax = qmax;
        p.out = out;
        p.ldo = ldo;
        int sms = 0;
        check_device(&sms);
        const int pairs = (int)((max_seq + 2 * mkq::attnpp::kBQ - 1) / (2 * mkq::attnpp::kBQ));
        const int64_t nitems = (int64_t)batch * heads * pairs;
        if (nitems > (1ll << 30)) return fail(MKQ_ERR_SHAPE, "too many attention work items");
        const int grid = (int)(nitems < sms ? nitems : sms);   // persistent, 1 CTA per SM
        launch_k(kern, dim3(grid), dim3(mkq::attnpp::kThreads), mkq::attnpp::kSmem, st, 1, mq, mkv, p, heads, pairs,
                 (int)nitems);
    } else {
    mkq::attn::Params p;
    p.qkv = static_cast<const __half*>(qkv);
    p.ld = ld;
    p.cu = cu;
    p.seq = (int)max_seq;
    p.hidden = (int)hidden;
    p.out_mode = out_mode;
    p.s_out = s_out;
    p.qmin = qmin;
    p.qmax = qmax;
    p.out = out;
    p.ldo = ldo;
    dim3 grid((unsigned)((max_seq + 63) / 64), (unsigned)heads, (unsigned)batch);
    launch_k(mkq::attn::flash_attn_kernel, grid, dim3(mkq::attn::kThreads), 0, st, 1, p);
    }
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "attention launch");
}

mkq_status mkq_attention_i8(const void* qkv, int64_t ld, int64_t batch, int64_t max_seq, const int32_t* cu,
                            int64_t tokens, int heads, int head_dim, float s_qkv, int out_mode, float s_out, int qmin,
                            int qmax, void* out, int64_t ldo, void* stream) {
    if (batch < 0 || max_seq < 0 || tokens < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (batch == 0 || tokens == 0) return MKQ_OK;
    if (!qkv || !out) return fail(MKQ_ERR_NULL, "qkv and out are required");
    if (head_dim != 64) return fail(MKQ_ERR_SHAPE, "head_dim must be 64");
    if (heads <= 0 || heads > 65535) return fail(MKQ_ERR_SHAPE, "heads out of range");
    if (max_seq <= 0 || max_seq > mkq::attn8::kMaxL) return fail(MKQ_ERR_SHAPE, "max_seq must be in [1, 128]");
    if (batch > 65535) return fail(MKQ_ERR_SHAPE, "batch must be <= 65535");
    if (!cu && tokens != batch * max_seq) return fail(MKQ_ERR_SHAPE, "tokens != batch*max_seq without cu_seqlens");
    const int64_t hidden = (int64_t)heads * 64;
    if (ld < 3 * hidden) return fail(MKQ_ERR_SHAPE, "ld_qkv smaller than 3*hidden bytes");
    if (!aligned16(qkv) || ld % 16) return fail(MKQ_ERR_ALIGN, "qkv rows must be 16-byte aligned");
    int64_t orow;
    if (out_mode == MKQ_OUT_F32) orow = 4 * hidden;
    else if (out_mode == MKQ_OUT_I4) orow = hidden / 2;
    else if (out_mode == MKQ_OUT_I8) orow = hidden;
    else return fail(MKQ_ERR_RANGE, "attention out_mode must be F32, I4 or I8");
    if (ldo < orow) return fail(MKQ_ERR_SHAPE, "ldo smaller than a row");
    if (!aligned16(out) || ldo % 16) return fail(MKQ_ERR_ALIGN, "out rows must be 16-byte aligned");
    if (!finite_pos(s_qkv)) return fail(MKQ_ERR_SCALE, "s_qkv must be > 0 and finite");
    if (out_mode != MKQ_OUT_F32) {
        if (!finite_pos(s_out)) return fail(MKQ_ERR_SCALE, "s_out must be > 0 and finite");
        if (!code_range_ok(out_mode == MKQ_OUT_I4 ? 4 : 8, qmin, qmax)) return fail(MKQ_ERR_RANGE, "qmin/qmax");
    }
    mkq_status s = check_device();
    if (s != MKQ_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PdlScope pdl_scope(tokens);
    mkq::attn8::Params p;
    p.qkv = static_cast<const int8_t*>(qkv);
    p.ld = ld;
    p.cu = cu;
    p.seq = (int)max_seq;
    p.hidden = (int)hidden;
    p.s = s_qkv;
    p.out_mode = out_mode;
    p.s_out = s_out;
    p.qmin = qmin;
    p.qmax = qmax;
    p.out = out;
    p.ldo = ldo;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(mkq::attn8::attn_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             mkq::attn8::kSmem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(attn_i8)");
        attr_set[dev] = true;
    }
    launch_k(mkq::attn8::attn_i8_kernel, dim3((unsigned)heads, (unsigned)batch, (unsigned)((max_seq + 63) / 64)),
             dim3(mkq::attn8::kThreads),
             mkq::attn8::kSmem, st, 1, p);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "attention_i8 launch");
}

mkq_status mkq_residual_layernorm(const float* x, const float* res, int64_t rows, int64_t cols, int64_t ld,
                                  const float* g, const float* b, float eps, float* y, int bits, float s_q,
                                  int qmin, int qmax, void* q, int64_t ldq, void* stream) {
    if (rows < 0 || cols < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (rows == 0) return MKQ_OK;
    if (!x || !g || !b || !y) return fail(MKQ_ERR_NULL, "x, g, b and y are required");
    if (bits && !q) return fail(MKQ_ERR_NULL, "q is required when bits != 0");
    if (cols <= 0 || cols % 4 || cols > 8192) return fail(MKQ_ERR_SHAPE, "cols must be a multiple of 4 in [4, 8192]");
    if (ld < cols || ld % 4) return fail(MKQ_ERR_SHAPE, "ld must be >= cols and a multiple of 4");
    if (!aligned16(x) || !aligned16(y) || !aligned16(g) || !aligned16(b) || (res && !aligned16(res)))
        return fail(MKQ_ERR_ALIGN, "x, res, y, g, b must be 16-byte aligned");
    if (!(eps >= 0.0f) || !std::isfinite(eps)) return fail(MKQ_ERR_SCALE, "eps must be finite and >= 0");
    if (bits) {
        if (bits != 4 && bits != 8) return fail(MKQ_ERR_RANGE, "bits must be 0, 4 or 8");
        if (!finite_pos(s_q)) return fail(MKQ_ERR_SCALE, "s_q must be > 0 and finite");
        if (!code_range_ok(bits, qmin, qmax)) return fail(MKQ_ERR_RANGE, "qmin/qmax");
        if (ldq < (bits == 4 ? cols / 2 : cols)) return fail(MKQ_ERR_SHAPE, "ldq too small");
        if ((reinterpret_cast<uintptr_t>(q) & 3) || ldq % 4) return fail(MKQ_ERR_ALIGN, "q must be 4-byte aligned");
    }
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int gr = grid_for(rows * 32, 256, sms);
    PdlScope pdl_scope(rows);
    uint8_t* qq = static_cast<uint8_t*>(q);
    const int ci = (int)cols;
    if (cols <= 1024 && rows <= 16384) launch_k(mkq::residual_ln_kernel<8, true>, dim3(gr), dim3(256), 0, st, 1, x, res, rows, ci, ld, g, b, eps, y, bits, s_q, qmin, qmax, qq, ldq);
    else if (cols <= 1024) launch_k(mkq::residual_ln_kernel<8>, dim3(gr), dim3(256), 0, st, 1, x, res, rows, ci, ld, g, b, eps, y, bits, s_q, qmin, qmax, qq, ldq);
    else if (cols <= 2048) launch_k(mkq::residual_ln_kernel<16>, dim3(gr), dim3(256), 0, st, 1, x, res, rows, ci, ld, g, b, eps, y, bits, s_q, qmin, qmax, qq, ldq);
    else launch_k(mkq::residual_ln_kernel<64>, dim3(gr), dim3(256), 0, st, 1, x, res, rows, ci, ld, g, b, eps, y, bits, s_q, qmin, qmax, qq, ldq);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "layernorm launch");
}

mkq_status mkq_interleave_blocks(const void* src, void* dst, int64_t g, int64_t rows, int64_t cb, int64_t ldd,
                                 void* stream) {
    if (g < 0 || rows < 0 || cb < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (g == 0 || rows == 0 || cb == 0) return MKQ_OK;
    if (!src || !dst) return fail(MKQ_ERR_NULL, "src and dst are required");
    if (cb % 16 || ldd < g * cb || ldd % 16) return fail(MKQ_ERR_SHAPE, "cb % 16, ld_dst >= g*cb, ld_dst % 16");
    if (!aligned16(src) || !aligned16(dst)) return fail(MKQ_ERR_ALIGN, "src/dst must be 16-byte aligned");
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    const int gr = grid_for(g * rows * (cb / 16), 256, sms);
    mkq::interleave_blocks_kernel<<<gr, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), g, rows, cb, ldd);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "interleave launch");
}

// ------------------------------------------------------------------ QAT / calibration
static constexpr int kQatMaxBlocks = 2048;

size_t mkq_fake_quant_workspace_size(int64_t) { return kQatMaxBlocks * sizeof(mkq::qat::Partial); }

mkq_status mkq_fake_quant(const float* x, int64_t n, const float* scale, int qmin, int qmax, float* y,
                          const float* grad_y, float* grad_x, double* grad_s, void* ws, size_t ws_bytes,
                          void* stream) {
    if (n < 0) return fail(MKQ_ERR_SHAPE, "negative n");
    if (!scale || (n > 0 && !x)) return fail(MKQ_ERR_NULL, "x and scale are required");
    if (grad_x && !grad_y) return fail(MKQ_ERR_NULL, "grad_x needs grad_y");
    if (!ws) return fail(MKQ_ERR_NULL, "a workspace is required");
    if (n > (int64_t(1) << 40)) return fail(MKQ_ERR_SHAPE, "n too large");
    if (ws_bytes < mkq_fake_quant_workspace_size(n))
        return fail(MKQ_ERR_WORKSPACE, "workspace needs %zu bytes", mkq_fake_quant_workspace_size(n));
    if ((reinterpret_cast<uintptr_t>(grad_s) & 7) || (ws && (reinterpret_cast<uintptr_t>(ws) & 15)))
        return fail(MKQ_ERR_ALIGN, "grad_s 8-byte, ws 16-byte aligned");
    if (!code_range_ok(8, qmin, qmax)) return fail(MKQ_ERR_RANGE, "need -128 <= qmin < qmax <= 127");
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int vec = aligned16(x) && (!y || aligned16(y)) && (!grad_y || aligned16(grad_y)) &&
                    (!grad_x || aligned16(grad_x));
    int64_t blocks = ((n + 3) / 4 + mkq::qat::kThreads - 1) / mkq::qat::kThreads;
    const int64_t cap = std::min<int64_t>(kQatMaxBlocks, (int64_t)sms * 8);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (!y && !grad_x && !grad_s) return MKQ_OK;
    auto* part = static_cast<mkq::qat::Partial*>(ws);
    mkq::qat::fake_quant_grad_kernel<<<(int)blocks, mkq::qat::kThreads, 0, st>>>(
        x, n, scale, qmin, qmax, y, grad_y, grad_x, part, vec);
    if (grad_s)
        mkq::qat::fake_quant_finalize_kernel<<<1, mkq::qat::kThreads, 0, st>>>(part, (int)blocks, scale, grad_s);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "fake_quant launch");
}

size_t mkq_act_scale_workspace_size(void) { return mkq::calib::kWsBytes; }

mkq_status mkq_act_scale(const float* x, int64_t n, double p, float l_max, float* s_out, void* ws, size_t ws_bytes,
                         void* stream) {
    if (n < 0) return fail(MKQ_ERR_SHAPE, "negative n");
    if (!x || !s_out || !ws) return fail(MKQ_ERR_NULL, "x, s_out and ws are required");
    if (n == 0) return fail(MKQ_ERR_SHAPE, "empty input has no quantile");
    if (ws_bytes < mkq::calib::kWsBytes) return fail(MKQ_ERR_WORKSPACE, "workspace needs %zu bytes", mkq::calib::kWsBytes);
    if (reinterpret_cast<uintptr_t>(ws) & 15) return fail(MKQ_ERR_ALIGN, "ws must be 16-byte aligned");
    if (!(p >= 0.0 && p <= 1.0)) return fail(MKQ_ERR_RANGE, "p must be in [0, 1]");
    if (!finite_pos(l_max)) return fail(MKQ_ERR_SCALE, "l_max must be > 0 and finite");
    int sms = 0;
    mkq_status s = check_device(&sms);
    if (s != MKQ_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // index arithmetic of the definition (R6): pos = p (n-1), fp64
    const double pos = p * (double)(n - 1);
    const double flo = std::floor(pos);
    const unsigned long long lo = (unsigned long long)flo;
    const unsigned long long hi = std::min<unsigned long long>(lo + 1, (unsigned long long)(n - 1));
    const double frac = pos - flo;
    using namespace mkq::calib;
    auto* state = static_cast<State*>(ws);
    auto* hist = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 64);
    const int vec = aligned16(x);
    int64_t blocks = (n / (vec ? 4 : 1) + kThreads - 1) / kThreads;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sms * 4));   // 4 x 512 threads per SM
    init_kernel<<<1, kThreads, 0, st>>>(state, hist, lo, hi);
    hist_kernel<0><<<(int)blocks, kThreads, 0, st>>>(x, n, vec, state, hist);
    select_kernel<0><<<1, kThreads, 0, st>>>(state, hist);
    hist_kernel<1><<<(int)blocks, kThreads, 0, st>>>(x, n, vec, state, hist);
    select_kernel<1><<<1, kThreads, 0, st>>>(state, hist);
    hist_kernel<2><<<(int)blocks, kThreads, 0, st>>>(x, n, vec, state, hist);
    select_kernel<2><<<1, kThreads, 0, st>>>(state, hist);
    finalize_kernel<<<1, 1, 0, st>>>(state, frac, l_max, s_out);
    cudaError_t e = cudaPeekAtLastError();
    return e == cudaSuccess ? MKQ_OK : cuda_fail(e, "act_scale launch");
}

// ------------------------------------------------------------------ BERT layer
// Does the layer run its residual + LayerNorm stages fused into the GEMMs
// (mkq_gemm_residual_ln: W^A + LN1, W^2 + LN2)?  W4A4 layers with hidden in
// {256, 512, 768, 1024} and at least 4096 tokens (below that the small-M GEMM
// plans and the standalone LN kernels are faster).
static bool layer_fused_ln(const mkq_layer* L, int64_t T) {
    // >= 4096 tokens: the 2-CTA fused kernel; small M: the N-cluster kernel when
    // every cluster is co-resident (Table-2 BS 16); in between the small-M
    // GEMM plans and the standalone LN kernels
    return L->bits == 4 && L->hidden % 256 == 0 && L->hidden <= 1024 && (T >= 4096 || lnc_ok(T, L->hidden));
}

struct LayerWs {
    size_t codes_in, qkv, codes_oa, o, h1, codes_h1, codes_ffn2, f, ln, total;
};

static LayerWs layer_ws(const mkq_layer* L, int64_t T) {
    LayerWs w;
    const int64_t h = L->hidden, F = L->ffn;
    const int64_t cb = L->bits == 4 ? 1 : 2;   // code bytes per 2 elements
    const bool fused = layer_fused_ln(L, T);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
    w.codes_in = take((size_t)T * h * cb / 2);
    w.qkv = take((size_t)T * 3 * h * 2);
    w.codes_oa = take((size_t)T * h * cb / 2);
    w.o = fused ? 0 : take((size_t)T * h * 4);
    w.h1 = take((size_t)T * h * 4);
    w.codes_h1 = take((size_t)T * h * cb / 2);
    w.codes_ffn2 = take((size_t)T * F * cb / 2);
    w.f = fused ? 0 : take((size_t)T * h * 4);
    int sms = 148;
    if (fused && check_device(&sms) != MKQ_OK) sms = 148;
    w.ln = fused ? take(ln_ws_bytes(sms, (int)(h / 256))) : 0;
    w.total = off;
    return w;
}

int mkq_layer_fused_ln(const mkq_layer* L, int64_t tokens) { return L && layer_fused_ln(L, tokens) ? 1 : 0; }

size_t mkq_bert_layer_workspace_size(const mkq_layer* L, int64_t tokens) {
    if (!L || tokens < 0) return 0;
    return layer_ws(L, tokens).total;
}

mkq_status mkq_bert_layer(const mkq_layer* L, const float* h_in, int64_t batch, int64_t max_seq,
                          const int32_t* cu, int64_t T, float* h_out, void* ws, size_t ws_bytes, void* stream) {
    if (!L) return fail(MKQ_ERR_NULL, "layer description is NULL");
    if (batch < 0 || max_seq < 0 || T < 0) return fail(MKQ_ERR_SHAPE, "negative dimension");
    if (T == 0) return MKQ_OK;
    if (!h_in || !h_out || !ws) return fail(MKQ_ERR_NULL, "h_in, h_out and ws are required");
    if (!L->w_qkv || !L->w_o || !L->w_1 || !L->w_2 || !L->sw_qkv || !L->sw_o || !L->sw_1 || !L->sw_2 ||
        !L->ln1_g || !L->ln1_b || !L->ln2_g || !L->ln2_b)
        return fail(MKQ_ERR_NULL, "layer weights, scales and LN parameters are required");
    if (L->bits != 4 && L->bits != 8) return fail(MKQ_ERR_RANGE, "bits must be 4 or 8");
    if (L->hidden <= 0 || L->hidden % 64 || L->heads * 64 != L->hidden)
        return fail(MKQ_ERR_SHAPE, "hidden must equal heads*64");
    if (L->ffn <= 0 || L->ffn % 32) return fail(MKQ_ERR_SHAPE, "ffn must be a positive multiple of 32");
    if (!finite_pos(L->s_qkv_in) || !finite_pos(L->s_o_in) || !finite_pos(L->s_ffn1_in) || !finite_pos(L->s_ffn2_in))
        return fail(MKQ_ERR_SCALE, "activation scales must be > 0 and finite");
    if (!cu && T != batch * max_seq) return fail(MKQ_ERR_SHAPE, "tokens != batch*max_seq without cu_seqlens");
    if (L->int_attention != 0 && L->int_attention != 1) return fail(MKQ_ERR_RANGE, "int_attention must be 0 or 1");
    if (L->int_attention && !finite_pos(L->s_attn)) return fail(MKQ_ERR_SCALE, "s_attn must be > 0 and finite");
    if (L->int_attention && max_seq > 128) return fail(MKQ_ERR_SHAPE, "int_attention needs max_seq <= 128");
    if (L->in_codes && !aligned16(L->in_codes)) return fail(MKQ_ERR_ALIGN, "in_codes must be 16-byte aligned");
    if (L->out_codes) {
        if (L->out_bits != 4 && L->out_bits != 8) return fail(MKQ_ERR_RANGE, "out_bits must be 4 or 8");
        if (!finite_pos(L->s_out_codes)) return fail(MKQ_ERR_SCALE, "s_out_codes must be > 0 and finite");
        if (!aligned16(L->out_codes)) return fail(MKQ_ERR_ALIGN, "out_codes must be 16-byte aligned");
    }
    const LayerWs W = layer_ws(L, T);
    if (ws_bytes < W.total) return fail(MKQ_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, W.total);
    if (!aligned16(ws)) return fail(MKQ_ERR_ALIGN, "workspace must be 16-byte aligned");
    mkq_status s = check_device();
    if (s != MKQ_OK) return s;

    const int bits = L->bits;
    const int qlo = bits == 4 ? -8 : -128, qhi = bits == 4 ? 7 : 127;
    const int64_t h = L->hidden, F = L->ffn;
    const int64_t cbh = bits == 4 ? h / 2 : h;   // code bytes per hidden row
    const int64_t cbf = bits == 4 ? F / 2 : F;
    uint8_t* base = static_cast<uint8_t*>(ws);
    uint8_t* codes_in = base + W.codes_in;
    __half* qkv = reinterpret_cast<__half*>(base + W.qkv);
    uint8_t* codes_oa = base + W.codes_oa;
    float* o = reinterpret_cast<float*>(base + W.o);
    float* h1 = reinterpret_cast<float*>(base + W.h1);
    uint8_t* codes_h1 = base + W.codes_h1;
    uint8_t* codes_ffn2 = base + W.codes_ffn2;
    float* f = reinterpret_cast<float*>(base + W.f);
    auto gemm = bits == 4 ? mkq_gemm_w4a4 : mkq_gemm_w8a8;

    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int sms = 0;
    check_device(&sms);
#define MKQ_TRY(x)                       \
    do {                                 \
        mkq_status _s = (x);             \
        if (_s != MKQ_OK) return _s;     \
    } while (0)
    // a1: quantize the layer input (per-tensor static scale, by value), unless
    // the previous layer's LN2 already wrote these codes (in_codes)
    if (L->in_codes)
        codes_in = static_cast<uint8_t*>(const_cast<void*>(L->in_codes));
    else
        MKQ_TRY(quantize_internal(h_in, T, h, h, nullptr, L->s_qkv_in, 0, bits, qlo, qhi, codes_in, cbh, sms, st));
    // a2-a4: QKV projection -> fp16 q|k|v (R10)
    if (L->int_attention) {
        // NEXT(2): int8 q|k|v codes (Eq.1, s_attn, [-127,127]) -> integer attention core (R19)
        mkq_epilogue e_i8{MKQ_OUT_I8, 0, L->s_attn, -127, 127, nullptr};
        MKQ_TRY(gemm(codes_in, cbh, L->w_qkv, cbh, T, 3 * h, h, L->s_qkv_in, L->sw_qkv, L->b_qkv, &e_i8, qkv,
                     3 * h, nullptr, 0, stream));
        MKQ_TRY(mkq_attention_i8(qkv, 3 * h, batch, max_seq, cu, T, L->heads, 64, L->s_attn,
                                 bits == 4 ? MKQ_OUT_I4 : MKQ_OUT_I8, L->s_o_in, qlo, qhi, codes_oa, cbh, stream));
    } else {
        mkq_epilogue e_f16{MKQ_OUT_F16, 0, 1.0f, 0, 0, nullptr};
        MKQ_TRY(gemm(codes_in, cbh, L->w_qkv, cbh, T, 3 * h, h, L->s_qkv_in, L->sw_qkv, L->b_qkv, &e_f16, qkv,
                     3 * h * 2, nullptr, 0, stream));
        // a8: attention core, fused quantize of OA with s_o_in
        MKQ_TRY(mkq_attention(qkv, 3 * h, batch, max_seq, cu, T, L->heads, 64, bits == 4 ? MKQ_OUT_I4 : MKQ_OUT_I8,
                              L->s_o_in, qlo, qhi, codes_oa, cbh, stream));
    }
    const bool fused_ln = layer_fused_ln(L, T);
    void* ln_ws = base + W.ln;
    const size_t ln_bytes = fused_ln ? ln_ws_bytes(sms, (int)(h / 256)) : 0;
    mkq_epilogue e_f32{MKQ_OUT_F32, 0, 1.0f, 0, 0, nullptr};
    if (fused_ln) {
        // W^A projection + residual + LN1 -> h1 fp32 and its codes for FFN1, one kernel (NEXT(4))
        MKQ_TRY(mkq_gemm_residual_ln(codes_oa, cbh, L->w_o, cbh, T, h, h, L->s_o_in, L->sw_o, L->b_o, h_in, h,
                                     L->ln1_g, L->ln1_b, L->ln_eps, h1, h, 4, L->s_ffn1_in, qlo, qhi, codes_h1, cbh,
                                     ln_ws, ln_bytes, stream));
    } else {
        // W^A projection (+ b^A) -> fp32
        MKQ_TRY(gemm(codes_oa, cbh, L->w_o, cbh, T, h, h, L->s_o_in, L->sw_o, L->b_o, &e_f32, o, h * 4, nullptr, 0,
                     stream));
        // LN1(o + h) -> h1 fp32 and its codes for FFN1 (fused a1)
        MKQ_TRY(mkq_residual_layernorm(o, h_in, T, h, h, L->ln1_g, L->ln1_b, L->ln_eps, h1, bits, L->s_ffn1_in, qlo,
                                       qhi, codes_h1, cbh, stream));
    }
    // FFN1: GELU + requantize to the FFN2 input codes (a5, a6 fused)
    mkq_epilogue e_ffn1{bits == 4 ? MKQ_OUT_I4 : MKQ_OUT_I8, 1, L->s_ffn2_in, qlo, qhi, L->ffn1_requant_table};
    MKQ_TRY(gemm(codes_h1, cbh, L->w_1, cbh, T, F, h, L->s_ffn1_in, L->sw_1, L->b_1, &e_ffn1, codes_ffn2, cbf,
                 nullptr, 0, stream));
    const int ob = L->out_codes ? L->out_bits : 0;
    if (fused_ln) {
        // FFN2 + residual + LN2 -> h_out (+ the next layer's input codes), one kernel (NEXT(4))
        MKQ_TRY(mkq_gemm_residual_ln(codes_ffn2, cbf, L->w_2, cbf, T, h, F, L->s_ffn2_in, L->sw_2, L->b_2, h1, h,
                                     L->ln2_g, L->ln2_b, L->ln_eps, h_out, h, ob, ob ? L->s_out_codes : 1.0f,
                                     ob == 4 ? -8 : -128, ob == 4 ? 7 : 127, L->out_codes, ob == 4 ? h / 2 : h, ln_ws,
                                     ln_bytes, stream));
    } else {
        // FFN2 -> fp32
        MKQ_TRY(gemm(codes_ffn2, cbf, L->w_2, cbf, T, h, F, L->s_ffn2_in, L->sw_2, L->b_2, &e_f32, f, h * 4, nullptr,
                     0, stream));
        // LN2(f + h1) -> h_out (+ the next layer's input codes, fused a1)
        MKQ_TRY(mkq_residual_layernorm(f, h1, T, h, h, L->ln2_g, L->ln2_b, L->ln_eps, h_out, ob,
                                       ob ? L->s_out_codes : 1.0f, ob == 4 ? -8 : -128, ob == 4 ? 7 : 127,
                                       L->out_codes, ob == 4 ? h / 2 : h, stream));
    }
#undef MKQ_TRY
    return MKQ_OK;
}

}  // extern "C"
