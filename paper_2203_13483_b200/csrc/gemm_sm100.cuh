// gemm_sm100.cuh -- W4A4 / W8A8 GEMM with exact int32 accumulation on the
// sm_100a 5th-generation tensor cores (tcgen05.mma kind::i8, D in TMEM) and a
// fused dequant / GELU / requantize epilogue.  §8(a) rows a2-a7.
//
//   out[m, n] = epi( sum_k a[m, k] * w[n, k] )
//
// Operands are K-major ("TN"): A [M, K] activations, W [N, K] weights.
//
// W4A4 (kInt4): packed int4 tiles (two codes per byte, D2 layout) are
// TMA-loaded into a staging ring; four "unpack" warps expand them to int8 in
// the UMMA canonical K-major SWIZZLE_128B layout.  Blackwell has no integer
// int4 MMA; the unpack keeps the products exact (e2m1 FP4 cannot represent
// +-5, +-7, -8).  The expansion costs 3 ALU ops per 8 codes:
//     lo = (p << 4) & 0xF0F0F0F0     -> bytes 16*code[even k]
//     hi =  p       & 0xF0F0F0F0     -> bytes 16*code[odd  k]
// i.e. each int8 lane holds 16x the code (no sign-fix needed: the nibble
// already sits in the top half of the byte) and the K order inside a 32-byte
// MMA K-step is permuted identically for A and W.  Both operands carry the
// factor 16, so the s32 accumulator equals 256 * sum_k a*w exactly
// (|acc| <= 256*64*K < 2^31 for K <= 131040) and the epilogue recovers the
// true sum with an exact arithmetic shift (acc >> 8).
//
// W8A8: int8 tiles are TMA-loaded directly in the SWIZZLE_128B layout.
//
// Roles (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma (K=32 each) per 128-K block
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> dequant/GELU/requant -> global
//   warps 8-11  int4 -> int8 unpack (W4A4 only)
//   warp 3      (small-M plans) column scales / bias (/ LN gamma, beta) -> smem
// Pipelines: packed ring (TMA -> unpack), int8 ring (unpack|TMA -> MMA),
// double-buffered TMEM accumulators (MMA -> epilogue), so the epilogue of
// tile i overlaps the mainloop of tile i+1.
//
// Small-M plans (kCl: one tile per CTA, the paper's Table-2 regime):
//   * int4 (GemmCfg<BN, true, true>, kTA): 256-K stages; A is unpacked into
//     tensor memory (lane = row, tcgen05.st) by warps 8-11 and 4-7 (one half
//     of each stage each) and read by the MMA from there; W unpacks to the
//     SW128 ring.  BN 64 (K split over a cluster for long K) or 128.
//   * the unsplit epilogue stages 32-row blocks and TMA-stores them; the K
//     split reduces exact int32 partials over DSMEM first.
//   * kLnC (gemm_lnc_kernel): an N-cluster of N/64 CTAs per 128-row block adds
//     the residual and applies LayerNorm (+ Eq.1 codes) with row statistics
//     exchanged over DSMEM.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "epilogue.cuh"
#include "ptx.cuh"

namespace mkq {

enum OutMode : int { OUT_F32 = 0, OUT_BF16 = 1, OUT_I32 = 2, OUT_I4 = 3, OUT_I8 = 4, OUT_F16 = 5 };

struct EpiParams {
    int mode;
    int gelu;
    float s_a;
    const float* s_w;
    const float* bias;
    float s_out;
    int qmin, qmax;
    void* out;
    int64_t ldo_bytes;
};

template <int BN_, bool kInt4_, bool kSmall_ = false>
struct GemmCfg {
    static constexpr int BM = 128;
    static constexpr int BN = BN_;
    static constexpr bool kInt4 = kInt4_;
    // BN 64 int4 is the small-M plan (one tile per CTA, kTA): its A operand is
    // unpacked into tensor memory and read by the MMA from there (shared memory
    // carries the packed tiles and the unpacked W only), and a stage spans 256 K
    // (128-byte packed rows): at Table-2 sizes a stage's time is set by the
    // number of TMA rows in flight, not by bytes (int4 and int8 stages of 128 K
    // both took ~0.35 us with 4 stages in flight, tools/trace_small.py), so
    // 256-K int4 stages halve the time per K
    static constexpr bool kTA = kInt4 && kSmall_;   // (BN 64, or 128 for wider small-M tiles)
    static constexpr int BK = kTA ? 256 : 128;      // K elements per block (=128 int8 bytes/row otherwise)
    static constexpr int kA8 = kTA ? 0 : BM * BK;   // int8 bytes of A per stage (kTA: A lives in TMEM)
    static constexpr int kB8 = BN * BK;             // (kTA: BK/128 SW128 sub-tiles of BN x 128 B)
    static constexpr int kStage8 = kA8 + kB8;
    static constexpr int kAP = BM * BK / 2;         // packed bytes of A per stage
    static constexpr int kBP = BN * BK / 2;
    static constexpr int kStageP = kAP + kBP;
    static constexpr int S8 = kInt4 ? ((BN == 256 || (kTA && BN == 128)) ? 3 : 4) : 4;
    static constexpr int SP = kInt4 ? ((BN == 256 || (kTA && BN == 128)) ? 3 : 4) : 0;
    static_assert(BN == 64 || BN == 128 || BN == 256, "BN");
    static constexpr int kThreads = kInt4 ? 384 : 256;
    static constexpr uint32_t kTaCol = 128;         // first A column (kTA): accumulator in [0, 64)
    static constexpr uint32_t kTaStageCols = BK / 4;   // A columns per stage (4 K bytes per column)
    static constexpr uint32_t kTmemCols = kTA ? 512 : 2 * BN;   // (otherwise a double-buffered accumulator)
    static_assert(!kTA || kTaCol + S8 * kTaStageCols <= kTmemCols, "TMEM budget");
    static constexpr int kBarBytes = 8 * (2 * S8 + 2 * SP + 4) + 16;
    static constexpr int kSmem = 1024 + S8 * kStage8 + SP * kStageP + kBarBytes;
    static_assert(kSmem <= 232448, "shared memory budget");
};

// ------------------------------------------------------------------ epilogue store
// y (dequant [+GELU]) -> the output mode's encoding, one row, 32 columns.
__device__ __forceinline__ void epilogue_emit(const EpiParams& ep, float (&y)[32], uint8_t* orow, int n) {
    if (ep.gelu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) y[i] = gelu_pinned(y[i]);
    }
    switch (ep.mode) {
    case OUT_F32: {
        float4* o = reinterpret_cast<float4*>(orow + (int64_t)n * 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
        break;
    }
    case OUT_BF16:
    case OUT_F16: {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            w[i] = ep.mode == OUT_BF16 ? pack_bf16x2(y[2 * i], y[2 * i + 1]) : pack_f16x2(y[2 * i], y[2 * i + 1]);
        uint4* o = reinterpret_cast<uint4*>(orow + (int64_t)n * 2);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        break;
    }
    case OUT_I4: {
        // Eq.1 via the reciprocal; a group with a value near a rounding
        // boundary takes the exact division (quant_group_rcp, bit-identical)
        int q[32];
        quant_group_rcp(y, quant_rcp(ep.s_out, ep.qmin, ep.qmax), q);
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int q8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q8[j] = q[8 * i + j];
            w[i] = pack_nib8(q8);
        }
        *reinterpret_cast<uint4*>(orow + n / 2) = make_uint4(w[0], w[1], w[2], w[3]);
        break;
    }
    case OUT_I8: {
        int q[32];
        quant_group_rcp(y, quant_rcp(ep.s_out, ep.qmin, ep.qmax), q);   // (as OUT_I4)
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = pack_byte4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
        uint4* o = reinterpret_cast<uint4*>(orow + n);
        o[0] = make_uint4(w[0], w[1], w[2], w[3]);
        o[1] = make_uint4(w[4], w[5], w[6], w[7]);
        break;
    }
    default:
        break;
    }
}

// Exact int32 sums acc[32] of one row -> dequant (R4) with the per-column
// sc = fl(s_a s_w[n]) and bias read from `sc`/`bb` (global via __ldg, or
// shared memory), then the output encoding.
template <bool kSmemScales>
__device__ __forceinline__ void epilogue_acc(const EpiParams& ep, const int32_t (&acc)[32], int row, int n,
                                             const float* sc_s, const float* b_s) {
    uint8_t* orow = reinterpret_cast<uint8_t*>(ep.out) + (int64_t)row * ep.ldo_bytes;
    if (ep.mode == OUT_I32) {
        int4* o = reinterpret_cast<int4*>(orow + (int64_t)n * 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = make_int4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
        return;
    }
    float y[32];
    const bool hb = ep.bias != nullptr;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const float sc = kSmemScales ? sc_s[i] : __fmul_rn(ep.s_a, __ldg(ep.s_w + n + i));
        const float b = kSmemScales ? b_s[i] : (hb ? __ldg(ep.bias + n + i) : 0.0f);
        y[i] = dequant(acc[i], sc, b, hb);
    }
#ifdef MKQ_ABL_NOSTORE   // ablation (diagnostics only): no global stores
    if (y[0] != 1234.5f) return;
#endif
    epilogue_emit(ep, y, orow, n);
}

template <bool kInt4>
__device__ __forceinline__ void epilogue_store(const EpiParams& ep, const uint32_t (&v)[32], int row, int n) {
    int32_t acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = kInt4 ? ((int32_t)v[i] >> 8) : (int32_t)v[i];
    epilogue_acc<false>(ep, acc, row, n, nullptr, nullptr);
}

// Small-M direct epilogue: one row's 32 outputs (columns n..n+31) -> the
// TMA-store staging boxes of one warp (32 rows).  Box layout per output mode
// (make_out_map in mkq_abi.cu): f32/i32 two boxes of 16 columns (64 B rows,
// SWIZZLE_64B), f16/bf16 one of 32 columns (64 B, SWIZZLE_64B), i8 32 B rows
// (SWIZZLE_32B), i4 16 B rows (no swizzle); boxes are 2 KB apart.  Same
// arithmetic as epilogue_acc/epilogue_emit (R4, R7, R11, Eq.1).
__device__ __forceinline__ uint32_t stage_off(int r, int c, int P) {
    const int f = P == 64 ? ((r >> 1) & 3) : (P == 32 ? ((r >> 2) & 1) : 0);
    return (uint32_t)(r * P + ((c ^ f) << 4));
}
__device__ __forceinline__ int stage_boxes(int mode) { return mode == OUT_F32 || mode == OUT_I32 ? 2 : 1; }
__device__ __forceinline__ void epilogue_acc_stage(const EpiParams& ep, const int32_t (&acc)[32], const float* sc_s,
                                                   const float* b_s, uint8_t* stage, int r) {
    if (ep.mode == OUT_I32) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<int4*>(stage + (k >> 2) * 2048 + stage_off(r, k & 3, 64)) =
                make_int4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
        return;
    }
    float y[32];
    const bool hb = ep.bias != nullptr;
#pragma unroll
    for (int i = 0; i < 32; ++i) y[i] = dequant(acc[i], sc_s[i], b_s[i], hb);
    if (ep.gelu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) y[i] = gelu_pinned(y[i]);
    }
    switch (ep.mode) {
    case OUT_F32:
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4*>(stage + (k >> 2) * 2048 + stage_off(r, k & 3, 64)) =
                make_float4(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3]);
        break;
    case OUT_BF16:
    case OUT_F16: {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            w[i] = ep.mode == OUT_BF16 ? pack_bf16x2(y[2 * i], y[2 * i + 1]) : pack_f16x2(y[2 * i], y[2 * i + 1]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            *reinterpret_cast<uint4*>(stage + stage_off(r, k, 64)) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        break;
    }
    case OUT_I4: {
        // Eq.1 via the reciprocal; a group with a value near a rounding
        // boundary takes the exact division (quant_group_rcp, bit-identical)
        int q[32];
        quant_group_rcp(y, quant_rcp(ep.s_out, ep.qmin, ep.qmax), q);
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int q8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q8[j] = q[8 * i + j];
            w[i] = pack_nib8(q8);
        }
        *reinterpret_cast<uint4*>(stage + stage_off(r, 0, 16)) = make_uint4(w[0], w[1], w[2], w[3]);
        break;
    }
    case OUT_I8: {
        int q[32];
        quant_group_rcp(y, quant_rcp(ep.s_out, ep.qmin, ep.qmax), q);   // (as OUT_I4)
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = pack_byte4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
        *reinterpret_cast<uint4*>(stage + stage_off(r, 0, 32)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(stage + stage_off(r, 1, 32)) = make_uint4(w[4], w[5], w[6], w[7]);
        break;
    }
    default:
        break;
    }
}

#ifdef MKQ_TTRACE
// Diagnostics build only (tools/trace_small.py): per-CTA (globaltimer,
// clock64) at fixed points of the 1-CTA GEMM.
__device__ unsigned long long* g_ttrace = nullptr;
#define TTRACE(slot)                                                                        \
    do {                                                                                    \
        if (g_ttrace && blockIdx.x < 256) {                                                  \
            unsigned long long gt;                                                          \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));                          \
            g_ttrace[(blockIdx.x * 16 + (slot)) * 2] = gt;                                   \
            g_ttrace[(blockIdx.x * 16 + (slot)) * 2 + 1] = clock64();                        \
        }                                                                                   \
    } while (0)
#else
#define TTRACE(slot) \
    do {             \
    } while (0)
#endif

// Small-M fused W4A4 GEMM + residual + LayerNorm (+ Eq.1 codes) through an
// N-cluster (kLnC): the N/64 CTAs of one 128-row block form a thread-block
// cluster (N = 256..1024 -> 4..16 CTAs), each computes its 128 x 64 tile over
// the whole K, adds the residual (TMA, 32 x 32 fp32 SWIZZLE_128B boxes) and
// publishes per-row (mean, M2) of its 64 columns in shared memory; after a
// cluster barrier every CTA combines the N/64 partials of its rows over DSMEM
// in a fixed order (pairwise update: identical statistics in every CTA) and
// writes LN(r) and its codes with TMA stores.
struct LnCParams {
    CUtensorMap r, y, q;          // residual in; LN output fp32 (make_out_map F32); codes (I4/I8) or unused
    const float *g, *b;           // gamma, beta [N]
    float eps, s_q;
    int qbits, qmin, qmax;
};
constexpr int kLnCExtra = 1024 + 32768 + 1024 + 64;   // align slack, residual boxes, row statistics, barrier

// ------------------------------------------------------------------ kernel
template <class Cfg, bool kCl, bool kLnC>
__device__ __forceinline__ void gemm_i8tc_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmO,
                                               const EpiParams& ep, int M, int N, int K, int splits,
                                               const LnCParams* lp) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, S8 = Cfg::S8, SP = Cfg::SP;
    constexpr bool kInt4 = Cfg::kInt4;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring8 = smem;
    uint8_t* ringP = smem + S8 * Cfg::kStage8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ringP + SP * Cfg::kStageP);
    uint64_t* full8 = bars;
    uint64_t* empty8 = full8 + S8;
    uint64_t* fullP = empty8 + S8;
    uint64_t* emptyP = fullP + SP;
    uint64_t* tfull = emptyP + SP;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // kLnC: residual boxes [4 quadrants][2 column blocks] x 4 KB, row statistics, residual barrier
    uint8_t* lres = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tmem_slot) + 16 + 1023) & ~uintptr_t(1023));
    float2* lstat = reinterpret_cast<float2*>(lres + 32768);
    uint64_t* rbar = reinterpret_cast<uint64_t*>(lstat + Cfg::BM);
    static_assert(!kLnC || (kCl && Cfg::kTA && Cfg::BN == 64), "kLnC: small-M int4 plan, 64-column tiles");
    __shared__ float g_s[kLnC ? Cfg::BN : 1], be_s[kLnC ? Cfg::BN : 1];
    float rr[kLnC ? 64 : 1];   // kLnC epilogue: the row's residual sums r = y + res, across the cluster barrier

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) TTRACE(0);
    const int m_tiles = (M + BM - 1) / BM;
    const int n_tiles = (N + BN - 1) / BN;
    // Work units: (output tile, K split).  kCl (the small-M plan, SURVEY §8f
    // NEXT(1)): one unit per CTA, the `splits` CTAs of a thread-block cluster
    // share one output tile and each accumulates a K range; the exact int32
    // partials are staged in shared memory and reduce-scattered over DSMEM
    // (CTA r sums rows r*BM/splits.. of every peer -- integer addition, so
    // the result is exact in any order, R15) and all warps run the epilogue
    // of their row slice.  Otherwise (splits == 1) persistent over tiles.
    const int num_tiles = m_tiles * n_tiles * splits;
    const int nk = (K + Cfg::BK - 1) / Cfg::BK;
    auto k_range = [&](int unit, int& kb0, int& kb1) {
        const int ks = unit % splits;
        kb0 = (int)((int64_t)ks * nk / splits);
        kb1 = (int)((int64_t)(ks + 1) * nk / splits);
    };
    constexpr int kRP = Cfg::BN * 4 + 16;   // staged partial row pitch (bytes)
    static_assert(!kCl || Cfg::BM * kRP <= Cfg::S8 * Cfg::kStage8, "partial staging fits the int8 ring");
    __shared__ float sc_s[kCl ? Cfg::BN : 1], b_s[kCl ? Cfg::BN : 1];

    static_assert(!Cfg::kTA || kCl, "A in TMEM: one tile per CTA (small-M plan)");
    if (threadIdx.x == 0) {
        for (int i = 0; i < S8; ++i) {
            ptx::mbar_init(&full8[i], Cfg::kTA ? 8 : (kInt4 ? (kCl ? 32 : 128) : 1));
            ptx::mbar_init(&empty8[i], 1);
        }
        for (int i = 0; i < SP; ++i) {
            ptx::mbar_init(&fullP[i], 1);
            ptx::mbar_init(&emptyP[i], Cfg::kTA ? 8 : (kCl ? 32 : 128));
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 128);
        }
        if constexpr (kLnC) ptx::mbar_init(rbar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        if constexpr (kLnC) {
            ptx::tma_prefetch_desc(&lp->r);
            ptx::tma_prefetch_desc(&lp->y);
            if (lp->qbits) ptx::tma_prefetch_desc(&lp->q);
        }
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_launch();
    ptx::pdl_wait();
    if (threadIdx.x == 0) TTRACE(1);

    // Small-M plan, A in TMEM (kTA): the stage's unpack is split between two
    // warps per TMEM lane quadrant q (the unpack warp 8+q, half 0, and the
    // epilogue warp 4+q, half 1, which is idle until the accumulator is ready;
    // one warp per quadrant left a 256-K stage ~0.5 us of unpack latency).
    // Half h expands packed A chunks 4h..4h+3 of row 32q + lane (lane = row;
    // packed A arrives with the TMA 128-byte swizzle, so the lanes' row reads
    // are conflict-free) into TMEM columns 32h..32h+31 of the stage with one
    // tcgen05.st (column 8c..8c+3 = even codes of packed chunk c, 8c+4..8c+7 =
    // odd codes: the permutation W gets in shared memory), and W chunks 2h,
    // 2h+1 of each lane (rows 16q..16q+15) into the SW128 sub-tiles (K bytes
    // [128 t, 128 t + 128) in sub-tile t).
    auto ta_unpack = [&](int q, int h) {
        if constexpr (Cfg::kTA) {
            constexpr int kAC = Cfg::BK / 32;              // packed 16-byte chunks per row (8)
            constexpr int kBPer = (BN / 4) * kAC / 32;     // W chunks per lane (4 for BN 64, 8 for 128)
            constexpr int kBH = kBPer / 2;                 // per half
            static_assert(Cfg::BK == 256 && (BN == 64 || BN == 128), "kTA layout");
            int kb0, kb1;
            k_range(blockIdx.x, kb0, kb1);
            const int r = q * 32 + lane;
            const uint32_t aoff = (uint32_t)r * 128u, af = (uint32_t)r & 7u;
            const uint32_t lane_off = (uint32_t)(q * 32) << 16;
            for (int j = 0; kb0 + j < kb1; ++j) {
                const int sp = j % SP, s8 = j % S8;
                ptx::mbar_wait(&fullP[sp], (uint32_t)(j / SP) & 1u);
                ptx::mbar_wait(&empty8[s8], ((uint32_t)(j / S8) & 1u) ^ 1u);
                const uint32_t src = ptx::smem_u32(ringP + sp * Cfg::kStageP);
                uint4 pa[4], pb[kBH];
#pragma unroll
                for (int c = 0; c < 4; ++c) pa[c] = ptx::lds128(src + aoff + (((uint32_t)(4 * h + c) ^ af) << 4));
#pragma unroll
                for (int i = 0; i < kBH; ++i) {   // packed W arrives 128-byte swizzled as well
                    const int id = lane + 32 * (kBH * h + i);
                    const uint32_t rb = (uint32_t)((BN / 4) * q + id / kAC), cb = (uint32_t)(id % kAC);
                    pb[i] = ptx::lds128(src + Cfg::kAP + rb * 128u + ((cb ^ (rb & 7u)) << 4));
                }
                uint32_t w[32];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    ptx::unpack_i4x8(pa[cc].x, w[8 * cc + 0], w[8 * cc + 4]);
                    ptx::unpack_i4x8(pa[cc].y, w[8 * cc + 1], w[8 * cc + 5]);
                    ptx::unpack_i4x8(pa[cc].z, w[8 * cc + 2], w[8 * cc + 6]);
                    ptx::unpack_i4x8(pa[cc].w, w[8 * cc + 3], w[8 * cc + 7]);
                }
                ptx::tmem_st_32x32b_x32(tmem_base + lane_off + Cfg::kTaCol + Cfg::kTaStageCols * (uint32_t)s8 + 32u * (uint32_t)h, w);
                const uint32_t dst = ptx::smem_u32(ring8 + s8 * Cfg::kStage8 + Cfg::kA8);
#pragma unroll
                for (int i = 0; i < kBH; ++i) {
                    const int id = lane + 32 * (kBH * h + i);
                    const uint32_t rb = (uint32_t)((BN / 4) * q + id / kAC), cb = (uint32_t)(id % kAC);
                    const uint32_t sub = dst + (cb >> 2) * (uint32_t)(BN * 128) + rb * 128u, cl = cb & 3u;
                    uint4 lo, hi;
                    ptx::unpack_i4x8(pb[i].x, lo.x, hi.x);
                    ptx::unpack_i4x8(pb[i].y, lo.y, hi.y);
                    ptx::unpack_i4x8(pb[i].z, lo.z, hi.z);
                    ptx::unpack_i4x8(pb[i].w, lo.w, hi.w);
                    ptx::sts128(sub + (((2u * cl) ^ (rb & 7u)) << 4), lo);
                    ptx::sts128(sub + (((2u * cl + 1u) ^ (rb & 7u)) << 4), hi);
                }
                ptx::tmem_st_wait();             // this thread's A columns are written
                ptx::fence_proxy_async_smem();   // and its W bytes visible to the tensor core
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(&full8[s8]);
                    ptx::mbar_arrive(&emptyP[sp]);
                }
            }
        }
    };

    if (warp == 0) {
        // ---------------------------------------------------- TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int unit = blockIdx.x; unit < num_tiles; unit += gridDim.x) {
                const int tile = unit / splits;
                const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
                int kb0, kb1;
                k_range(unit, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    if constexpr (kInt4) {
                        ptx::mbar_wait(&emptyP[s], ph ^ 1);
                        uint8_t* dst = ringP + s * Cfg::kStageP;
                        ptx::mbar_arrive_expect_tx(&fullP[s], Cfg::kStageP);
                        ptx::tma_load_2d(&tmA, &fullP[s], dst, kb * (Cfg::BK / 2), m0);
                        ptx::tma_load_2d(&tmB, &fullP[s], dst + Cfg::kAP, kb * (Cfg::BK / 2), n0);
                        if (kb == kb0) TTRACE(2);
                        if (kb == kb0 + 4) TTRACE(3);
                        if (++s == SP) { s = 0; ph ^= 1; }
                    } else {
                        ptx::mbar_wait(&empty8[s], ph ^ 1);
                        uint8_t* dst = ring8 + s * Cfg::kStage8;
                        ptx::mbar_arrive_expect_tx(&full8[s], Cfg::kStage8);
                        ptx::tma_load_2d(&tmA, &full8[s], dst, kb * Cfg::BK, m0);
                        ptx::tma_load_2d(&tmB, &full8[s], dst + Cfg::kA8, kb * Cfg::BK, n0);
                        if (++s == S8) { s = 0; ph ^= 1; }
                    }
                }
            }
            if constexpr (kLnC) {   // the tile's residual: 8 boxes of 32 rows x 32 columns
                const int tile = blockIdx.x;
                const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
                ptx::mbar_arrive_expect_tx(rbar, 32768);
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    ptx::tma_load_2d(&lp->r, rbar, lres + b * 4096, n0 + 32 * (b & 1), m0 + 32 * (b >> 1));
            }
            if constexpr (!kInt4) {   // tail: the MMA's last commits on empty8 have landed
                for (int i = 0; i < S8; ++i) {
                    ptx::mbar_wait(&empty8[s], ph ^ 1);
                    if (++s == S8) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------- MMA issuer
        // Whole warp converged; elect.sync inside the MMA/commit wrappers.
        {
            constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
            const uint64_t dA0 = ptx::desc_sw128_kmajor(ptx::smem_u32(ring8));
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int unit = blockIdx.x; unit < num_tiles; unit += gridDim.x, ++it) {
                const int ab = it & 1;
                const uint32_t aph = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[ab], aph ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + ab * BN;
                int kb0, kb1;
                k_range(unit, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full8[s], ph);
                    ptx::tc_fence_after();
                    if (lane == 0 && kb == kb0) TTRACE(4);
                    if (lane == 0 && kb == kb1 - 1) TTRACE(5);
                    if (lane == 0 && kb > kb0 && kb - kb0 < 7) TTRACE(9 + kb - kb0);
                    const uint64_t da = dA0 + (uint64_t)((s * Cfg::kStage8) >> 4);
                    const uint64_t db = da + (uint64_t)(Cfg::kA8 >> 4);
                    if constexpr (Cfg::kTA) {   // A stage s in TMEM: 8 columns per 32-byte K step;
                        // W: K step k in SW128 sub-tile k/4 (BN x 128 B each), 32 B apart inside it
                        const uint32_t ta = tmem_base + Cfg::kTaCol + Cfg::kTaStageCols * (uint32_t)s;
#pragma unroll
                        for (int k = 0; k < Cfg::BK / 32; ++k)
                            ptx::mma_i8_ts_warp(d, ta + 8u * k, db + (uint64_t)((k >> 2) * ((BN * 128) >> 4) + 2 * (k & 3)),
                                                idesc, (kb != kb0) || k != 0);
                    } else {
#pragma unroll
                    for (int k = 0; k < Cfg::BK / 32; ++k)
                        ptx::mma_i8_ss_warp(d, da + 2 * k, db + 2 * k, idesc, (kb != kb0) || k != 0);
                    }
                    ptx::mma_commit_warp(&empty8[s]);
                    if (++s == S8) { s = 0; ph ^= 1; }
                }
                ptx::mma_commit_warp(&tfull[ab]);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------------------------------------------- epilogue
        const int q = warp & 3;   // TMEM lane quadrant owned by this warp
        if constexpr (Cfg::kTA) ta_unpack(q, 1);   // the mainloop's second unpack half first
        int it = 0;
        for (int unit = blockIdx.x; unit < num_tiles; unit += gridDim.x, ++it) {
            const int tile = unit / splits;
            const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
            const int ab = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            ptx::mbar_wait(&tfull[ab], aph);
            ptx::tc_fence_after();
            if (threadIdx.x == 128) TTRACE(6);
            const int row = m0 + q * 32 + lane;
            // kLnC: both 32-column blocks unrolled (rr is indexed statically: registers)
#pragma unroll
            for (int j = 0; j < (kLnC ? BN / 32 : 1); ++j) {
              if constexpr (kLnC) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + ab * BN + 32 * j, v);
                ptx::tmem_ld_wait();
                    // r = dequant(acc) + res for this row's 32 columns of block j (R4, R9)
                    if (j == 0) {
                        ptx::named_bar_sync(1, 160);
                        ptx::mbar_wait(rbar, 0);
                    }
                    const uint32_t bx = ptx::smem_u32(lres + (q * 2 + j) * 4096) + (uint32_t)lane * 128u;
                    const bool hb = ep.bias != nullptr;
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        float4 rs;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(rs.x), "=f"(rs.y), "=f"(rs.z), "=f"(rs.w)
                                     : "r"(bx + (uint32_t)((c4 ^ (lane & 7)) << 4)));
                        const float rv[4] = {rs.x, rs.y, rs.z, rs.w};
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int i = 4 * c4 + t;
                            const int32_t a = kInt4 ? ((int32_t)v[i] >> 8) : (int32_t)v[i];
                            rr[32 * j + i] = __fadd_rn(dequant(a, sc_s[32 * j + i], b_s[32 * j + i], hb), rv[t]);
                        }
                    }
                    if (j == 1) {   // this CTA's (mean, M2) of the row over its 64 columns
                        // 8 independent partial sums (no 64-long dependent chain), fixed order
                        float ps[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) ps[k] = rr[k];
#pragma unroll
                        for (int i = 8; i < 64; ++i) ps[i & 7] = __fadd_rn(ps[i & 7], rr[i]);
                        const float sum = __fadd_rn(__fadd_rn(__fadd_rn(ps[0], ps[1]), __fadd_rn(ps[2], ps[3])),
                                                    __fadd_rn(__fadd_rn(ps[4], ps[5]), __fadd_rn(ps[6], ps[7])));
                        const float mean = sum / 64.0f;   // IEEE; an exact multiply by 2^-6
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const float d = __fsub_rn(rr[k], mean);
                            ps[k] = __fmul_rn(d, d);
                        }
#pragma unroll
                        for (int i = 8; i < 64; ++i) {
                            const float d = __fsub_rn(rr[i], mean);
                            ps[i & 7] = __fmaf_rn(d, d, ps[i & 7]);
                        }
                        const float m2 = __fadd_rn(__fadd_rn(__fadd_rn(ps[0], ps[1]), __fadd_rn(ps[2], ps[3])),
                                                   __fadd_rn(__fadd_rn(ps[4], ps[5]), __fadd_rn(ps[6], ps[7])));
                        lstat[q * 32 + lane] = make_float2(mean, m2);
                    }
              }
            }
#pragma unroll 1
            for (int j = 0; j < (kLnC ? 0 : BN / 32); ++j) {
                const int n = n0 + 32 * j;
                if (n >= N) break;
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + ab * BN + 32 * j, v);
                ptx::tmem_ld_wait();
                if constexpr (kCl) {
                  if (splits == 1) {
                    // no K split: epilogue straight from TMEM (no cluster
                    // barrier, no DSMEM round trip); scales/bias staged by warp 3
                    // Rows are staged in the idle int8 ring (every MMA of this
                    // CTA's only tile has completed) and TMA-stored per warp: a
                    // row-per-lane STG scatters 32 rows per instruction and cost
                    // ~2 us per tile at Table-2 sizes (tools/trace_small.py).
                    if (j == 0) ptx::named_bar_sync(1, 160);
                    if (threadIdx.x == 128 && j == 0) TTRACE(8);
                    int32_t acc[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = kInt4 ? ((int32_t)v[i] >> 8) : (int32_t)v[i];
                    uint8_t* stage = ring8 + (q * (BN / 32) + j) * 4096;
                    epilogue_acc_stage(ep, acc, sc_s + 32 * j, b_s + 32 * j, stage, lane);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int y0 = m0 + q * 32;
                        if (ep.mode == OUT_F32 || ep.mode == OUT_I32) {
                            ptx::tma_store_2d(&tmO, stage, n, y0);
                            ptx::tma_store_2d(&tmO, stage + 2048, n + 16, y0);
                        } else {
                            ptx::tma_store_2d(&tmO, stage, ep.mode == OUT_I4 ? n / 2 : n, y0);
                        }
                        ptx::tma_store_commit();
                    }
                    if (threadIdx.x == 128 && j == 0) TTRACE(15);
                  } else {
                    // stage the (shifted) partial of row q*32+lane in the idle int8 ring
                    uint8_t* dst = ring8 + (q * 32 + lane) * kRP + j * 128;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        uint4 t;
                        t.x = kInt4 ? (uint32_t)((int32_t)v[4 * i] >> 8) : v[4 * i];
                        t.y = kInt4 ? (uint32_t)((int32_t)v[4 * i + 1] >> 8) : v[4 * i + 1];
                        t.z = kInt4 ? (uint32_t)((int32_t)v[4 * i + 2] >> 8) : v[4 * i + 2];
                        t.w = kInt4 ? (uint32_t)((int32_t)v[4 * i + 3] >> 8) : v[4 * i + 3];
                        *reinterpret_cast<uint4*>(dst + 16 * i) = t;
                    }
                  }
                } else if (row < M) {
                    epilogue_store<kInt4>(ep, v, row, n);
                }
            }
            if (kCl && splits == 1 && lane == 0) ptx::tma_store_wait_read<0>();   // staging is read before exit
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[ab]);
            if (threadIdx.x == 128) TTRACE(7);
        }
    } else if (kCl && warp == 3) {
        // ---------------------------------------------------- scale/bias prefetch
        const int n0 = ((blockIdx.x / splits) % n_tiles) * BN;
        for (int c = lane; c < BN; c += 32) {
            const int n = n0 + c;
            sc_s[c] = n < N ? __fmul_rn(ep.s_a, __ldg(ep.s_w + n)) : 0.0f;
            b_s[c] = (n < N && ep.bias) ? __ldg(ep.bias + n) : 0.0f;
            if constexpr (kLnC) {
                g_s[c] = n < N ? __ldg(lp->g + n) : 0.0f;
                be_s[c] = n < N ? __ldg(lp->b + n) : 0.0f;
            }
        }
        if (splits == 1) ptx::named_bar_arrive(1, 160);   // -> the epilogue warps
    } else if (kInt4 && warp >= 8) {
        // ---------------------------------------------------- int4 -> int8 unpack
        const int u = threadIdx.x - 256;
        constexpr int kChunks = (BM + BN) * (Cfg::BK / 32);   // 16-byte packed chunks / stage
        static_assert(kChunks % 128 == 0, "chunk split");
        if constexpr (Cfg::kTA) {
            ta_unpack(warp - 8, 0);
            // tail: the last MMA commit on slot q has landed
            const int q = warp - 8;
            int kb0, kb1;
            k_range(blockIdx.x, kb0, kb1);
            const int n = kb1 - kb0;
            if (q < n && q < S8) {
                const int jl = ((n - 1 - q) / S8) * S8 + q;
                ptx::mbar_wait(&empty8[q], (uint32_t)(jl / S8) & 1u);
            }
        } else {
        int sp = 0, s8 = 0;
        uint32_t php = 0, ph8 = 0;
        for (int unit = blockIdx.x; unit < num_tiles; unit += gridDim.x) {
            int kb0, kb1;
            k_range(unit, kb0, kb1);
            for (int kb = kb0; kb < kb1; ++kb) {
                ptx::mbar_wait(&fullP[sp], php);
                ptx::mbar_wait(&empty8[s8], ph8 ^ 1);
                const uint8_t* src = ringP + sp * Cfg::kStageP;
                uint8_t* dst = ring8 + s8 * Cfg::kStage8;
#pragma unroll 4
                for (int i = 0; i < kChunks / 128; ++i) {
                    const int id = u + 128 * i;
                    const int r = id >> 2, c = id & 3;
                    const uint4 p = *reinterpret_cast<const uint4*>(src + r * 64 + c * 16);
                    uint4 lo, hi;
                    lo.x = (p.x << 4) & 0xF0F0F0F0u; hi.x = p.x & 0xF0F0F0F0u;
                    lo.y = (p.y << 4) & 0xF0F0F0F0u; hi.y = p.y & 0xF0F0F0F0u;
                    lo.z = (p.z << 4) & 0xF0F0F0F0u; hi.z = p.z & 0xF0F0F0F0u;
                    lo.w = (p.w << 4) & 0xF0F0F0F0u; hi.w = p.w & 0xF0F0F0F0u;
                    const int r7 = r & 7;
                    uint8_t* drow = dst + r * 128;
                    *reinterpret_cast<uint4*>(drow + (((2 * c) ^ r7) << 4)) = lo;
                    *reinterpret_cast<uint4*>(drow + (((2 * c + 1) ^ r7) << 4)) = hi;
                }
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&full8[s8]);
                ptx::mbar_arrive(&emptyP[sp]);
                if (++sp == SP) { sp = 0; php ^= 1; }
                if (++s8 == S8) { s8 = 0; ph8 ^= 1; }
            }
        }
        for (int i = 0; i < S8; ++i) {   // tail: the MMA's last commits on empty8 have landed
            ptx::mbar_wait(&empty8[s8], ph8 ^ 1);
            if (++s8 == S8) { s8 = 0; ph8 ^= 1; }
        }
        }
    }

    if constexpr (kLnC) {
        // pass 2: the row statistics of all N/64 CTAs of the cluster (DSMEM,
        // fixed order, pairwise update), LN(r) -> staged boxes -> TMA stores
        if (threadIdx.x == 128) TTRACE(12);
        ptx::cluster_sync();   // every CTA's lstat is written and visible
        if (threadIdx.x == 128) TTRACE(13);
        if (warp >= 4 && warp < 8) {
            const int q = warp & 3;
            const int tile = blockIdx.x;
            const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
            const int rl = q * 32 + lane;
            const uint32_t sa = ptx::smem_u32(lstat + rl);
            // all peers' partials in flight at once (<= 16 CTAs; a dependent
            // DSMEM round trip per peer cost ~0.18 us each, tools/trace_small.py)
            float2 part[16];
#pragma unroll
            for (int pc = 0; pc < 16; ++pc) {
                if (pc < n_tiles) {
                    uint32_t ra;
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sa), "r"(pc));
                    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(part[pc].x), "=f"(part[pc].y) : "r"(ra));
                }
            }
            // this CTA is done reading its peers: release them early (the matching
            // wait is the last thing before exit)
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            float mean = 0.0f, M2 = 0.0f;
#pragma unroll
            for (int pc = 0; pc < 16; ++pc) {
                if (pc >= n_tiles) break;
                const float2 o = part[pc];
                if (pc == 0) {
                    mean = o.x;
                    M2 = o.y;
                } else {   // equal counts 64: Chan et al.'s pairwise update
                    // (pc is a compile-time constant in the unrolled loop: both IEEE
                    // quotients fold to constants instead of a dependent division chain)
                    const float d = __fsub_rn(o.x, mean);
                    const float nt = (float)(64 * (pc + 1)), nw = (float)(64 * pc);
                    mean = __fadd_rn(mean, __fmul_rn(d, 64.0f / nt));
                    M2 = __fadd_rn(__fadd_rn(M2, o.y), __fmul_rn(__fmul_rn(d, d), (nw * 64.0f) / nt));
                }
            }
            const float rstd = rsqrtf(__fadd_rn(__fdiv_rn(M2, (float)N), lp->eps));
            if (threadIdx.x == 128) TTRACE(14);
            const QuantRcp Qr = quant_rcp(lp->s_q, lp->qmin, lp->qmax);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                uint8_t* stage = ring8 + (q * 2 + j) * 8192;   // y: 2 x 2 KB (16 columns, SW64); codes at +4 KB
                float o[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int c = 32 * j + i;
                    o[i] = __fmaf_rn(__fmul_rn(__fsub_rn(rr[c], mean), rstd), g_s[c], be_s[c]);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    *reinterpret_cast<float4*>(stage + (k >> 2) * 2048 + stage_off(lane, k & 3, 64)) =
                        make_float4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
                if (lp->qbits == 4) {
                    uint32_t w[4];
                    bool near = false;
#pragma unroll
                    for (int g8 = 0; g8 < 4; ++g8) {
                        float v8[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) v8[t] = o[8 * g8 + t];
                        w[g8] = quant_nib8_fast(v8, Qr, near);
                    }
                    if (__builtin_expect(near, 0)) {
#pragma unroll
                        for (int g8 = 0; g8 < 4; ++g8)
                            w[g8] = quant_nib8_exact(o[8 * g8], o[8 * g8 + 1], o[8 * g8 + 2], o[8 * g8 + 3], o[8 * g8 + 4],
                                                     o[8 * g8 + 5], o[8 * g8 + 6], o[8 * g8 + 7], lp->s_q, lp->qmin,
                                                     lp->qmax);
                    }
                    *reinterpret_cast<uint4*>(stage + 4096 + stage_off(lane, 0, 16)) = make_uint4(w[0], w[1], w[2], w[3]);
                } else if (lp->qbits == 8) {
                    uint32_t w[8];
#pragma unroll
                    for (int g4 = 0; g4 < 8; ++g4) w[g4] = quant_byte4_rcp(o[4 * g4], o[4 * g4 + 1], o[4 * g4 + 2], o[4 * g4 + 3], Qr);
                    *reinterpret_cast<uint4*>(stage + 4096 + stage_off(lane, 0, 32)) = make_uint4(w[0], w[1], w[2], w[3]);
                    *reinterpret_cast<uint4*>(stage + 4096 + stage_off(lane, 1, 32)) = make_uint4(w[4], w[5], w[6], w[7]);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int n = n0 + 32 * j, y0 = m0 + q * 32;
                    ptx::tma_store_2d(&lp->y, stage, n, y0);
                    ptx::tma_store_2d(&lp->y, stage + 2048, n + 16, y0);
                    if (lp->qbits) ptx::tma_store_2d(&lp->q, stage + 4096, lp->qbits == 4 ? n / 2 : n, y0);
                    ptx::tma_store_commit();
                }
            }
            if (threadIdx.x == 128) TTRACE(15);
            if (lane == 0) ptx::tma_store_wait_read<0>();   // staging read before exit
        } else {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        }
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // peers have read this CTA's lstat
    }
    if constexpr (kCl && Cfg::BN == 64) if (splits > 1) {   // (wider small-M tiles run unsplit)
        // DSMEM reduce-scatter of the staged partials + epilogue (all warps)
        ptx::cluster_sync();   // release/acquire: every peer's staged rows are visible
        const int tile = blockIdx.x / splits;
        const int m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
        const int rank = (int)ptx::cluster_ctarank();
        // CTA `rank` owns the 32-row groups grp = rank, rank + splits, ... of
        // the tile; one warp per (group, 32-column block): lane = row, sums
        // the peers' partials over DSMEM, stages the outputs and TMA-stores
        // them (warp-private 4 KB staging slot past the partials)
        constexpr int kJ = BN / 32;
        const int ngroups = (min(BM, M - m0) + 31) / 32;
        const int owned = ngroups > rank ? (ngroups - rank + splits - 1) / splits : 0;
        const int nwarps = (int)(blockDim.x >> 5);
        const uint32_t red0 = ptx::smem_u32(ring8);
        static_assert(Cfg::BM * kRP <= 40960 &&
                          40960 + (Cfg::kThreads / 32) * 4096 <= Cfg::S8 * Cfg::kStage8 + Cfg::SP * Cfg::kStageP,
                      "partials + per-warp staging fit the idle rings (int8 ring, then the packed ring)");
        uint8_t* stage = ring8 + 40960 + warp * 4096;
        for (int u = warp; u < owned * kJ; u += nwarps) {
            const int grp = rank + splits * (u / kJ), j = u % kJ;
            const int rl = grp * 32 + lane, n = n0 + 32 * j;
            int32_t acc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = 0;
            // all 8 loads of a peer in flight before any add (in-order issue)
            for (int sp = 0; sp < splits; ++sp) {
                uint32_t ra;
                asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(red0 + rl * kRP + j * 128), "r"(sp));
                uint4 x[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(x[i].x), "=r"(x[i].y), "=r"(x[i].z), "=r"(x[i].w) : "r"(ra + 16 * i));
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    acc[4 * i] += (int32_t)x[i].x; acc[4 * i + 1] += (int32_t)x[i].y;
                    acc[4 * i + 2] += (int32_t)x[i].z; acc[4 * i + 3] += (int32_t)x[i].w;
                }
            }
            if (lane == 0) ptx::tma_store_wait_read<0>();   // this warp's previous store has read the slot
            __syncwarp();
            epilogue_acc_stage(ep, acc, sc_s + 32 * j, b_s + 32 * j, stage, lane);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                const int y0 = m0 + grp * 32;
                if (ep.mode == OUT_F32 || ep.mode == OUT_I32) {
                    ptx::tma_store_2d(&tmO, stage, n, y0);
                    ptx::tma_store_2d(&tmO, stage + 2048, n + 16, y0);
                } else {
                    ptx::tma_store_2d(&tmO, stage, ep.mode == OUT_I4 ? n / 2 : n, y0);
                }
                ptx::tma_store_commit();
            }
        }
        if (lane == 0) ptx::tma_store_wait_read<0>();
        if (threadIdx.x == 128) TTRACE(8);
        ptx::cluster_sync();   // peers may still be reading this CTA's rows
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TTRACE(9);
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

template <class Cfg, bool kCl = false>
__global__ void __launch_bounds__(Cfg::kThreads, 1)
    gemm_i8tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmO, const EpiParams ep, int M, int N, int K, int splits) {
    gemm_i8tc_body<Cfg, kCl, false>(tmA, tmB, tmO, ep, M, N, K, splits, nullptr);
}

// kLnC entry: one 128 x 64 tile per CTA, clusters of N/64 CTAs along N
template <class Cfg>
__global__ void __launch_bounds__(Cfg::kThreads, 1)
    gemm_lnc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ LnCParams lp, const EpiParams ep, int M, int N, int K) {
    gemm_i8tc_body<Cfg, true, true>(tmA, tmB, lp.y, ep, M, N, K, 1, &lp);
}

}  // namespace mkq
