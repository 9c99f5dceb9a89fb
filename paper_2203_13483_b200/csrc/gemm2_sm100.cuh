// gemm2_sm100.cuh -- W4A4 GEMM on a CTA pair (cta_group::2): the large-M
// path of mkq_gemm_w4a4 (§8a rows a2-a6).
//
// Same arithmetic as gemm_sm100.cuh (exact int32 accumulation of 16a x 16w,
// acc >> 8, pinned epilogue), re-tiled for the B200 tensor core:
//   * a cluster of 2 CTAs on one TPC computes a 256 x BN output tile with
//     tcgen05.mma.cta_group::2 (M = 256): each CTA stages 128 rows of A and
//     BN/2 rows of W, so the shared-memory traffic per MMA (TMA write +
//     unpack LDS/STS + tensor-core read) per SM is 2/3 of the 1-CTA
//     128 x 256 tile;
//   * 8 unpack warps per CTA (4 x 16-byte chunks per thread per stage, all
//     loads issued before any store);
//   * 8 epilogue warps per CTA (2 per TMEM lane quadrant, each half the
//     columns), per-tile scale/bias staged in shared memory, TMEM read in
//     16-column slices, and the exact y-space requant table (requant.cuh)
//     for the fused GELU + requantize output;
//   * double-buffered TMEM accumulators (2 x BN columns per CTA) so the
//     epilogue of tile i overlaps the mainloop of tile i+1.
// Barriers that gate the MMA (int8 stage full, accumulator empty) live in the
// leader CTA (rank 0) and collect one arrival per warp from both CTAs
// (fence.proxy.async + CTA-scope remote mbarrier arrive, as CUTLASS's 2-SM
// transform pipeline does; a cluster-scope release would be a GPU-scope
// membar); MMA completion is multicast to both CTAs' barriers.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "epilogue.cuh"
#include "gemm_sm100.cuh"
#include "ptx.cuh"
#include "requant.cuh"

namespace mkq {

// Fused residual + LayerNorm (+ Eq.1 quantize) epilogue (kLn, NEXT(4) fused
// glue): y = LN(dequant(acc) + res) over full rows of N = 256 np columns.
// The np CTA pairs of a "group" compute the np 256-column tiles of the same
// 256 rows at the same time and exchange per-row partial sums (mean, then the
// centred sum of squares) through global memory (workspace `stats`, arrival
// counters `flags`, zeroed by the launcher before every launch).
struct Ln2Params {
    const float* res;                 // residual [M, N] fp32, row stride ldr elements
    int64_t ldr;
    const float *g, *b;               // LN gamma / beta [N]
    float eps;
    float* y;                         // LN output [M, N] fp32, row stride ldy elements
    int64_t ldy;
    uint8_t* q;                       // optional Eq.1 codes of y (qbits 4|8; 0 = none)
    int64_t ldq;
    int qbits, qmin, qmax;
    float s_q;
    float* stats;                     // [groups][2 buffers][2 stages][np][256 rows]
    uint32_t* flags;                  // [groups][2][2] counters, 32-byte stride
    int np;                           // 256-column tiles per row = CTA pairs per group
};

struct Epi2Params {
    EpiParams e;
    const void* table;   // rq table (global) or null
    Ln2Params ln;        // kLn only
};

template <int BN_, int EPI_ = 8, int UNP_ = 8, bool LUT4_ = false, bool LN_ = false, int LNB_ = 2>
struct Gemm2Cfg {
    static constexpr bool kLn = LN_;                 // fused residual + LayerNorm epilogue
    static constexpr bool kRegSplit = LUT4_ || LN_;  // setmaxnreg per role
    static constexpr bool kLut4 = LUT4_;             // int4 output through the compact requant table
    static constexpr int BM = 128;                  // A rows per CTA (MMA M = 256 per pair)
    static constexpr int BN = BN_;                  // MMA N (per pair)
    static constexpr int BNH = BN / 2;              // W rows per CTA
    static constexpr int BK = 128;
    static constexpr int kA8 = BM * BK;
    static constexpr int kB8 = BNH * BK;
    static constexpr int kStage8 = kA8 + kB8;
    static constexpr int kAP = BM * BK / 2;
    static constexpr int kBP = BNH * BK / 2;
    static constexpr int kStageP = kAP + kBP;
    // kLn: LNB_ residual/output boxes per epilogue warp; two boxes (short K,
    // epilogue-bound) take smem from the rings, one box (long K) keeps them
    static constexpr int kBoxes = LNB_;
    static constexpr bool kSmallRing = LN_ && LNB_ * (4096 + 1024) * EPI_ > 48 * 1024;
    static constexpr int S8 = kSmallRing ? 3 : 4;
    static constexpr int SP = kSmallRing ? 2 : 3;
    static constexpr int kEpiWarps = EPI_;          // 8 or 16 (2 or 4 per TMEM lane quadrant)
    static constexpr int kUnpWarps = UNP_;          // 8 or 4
    static constexpr int kThreads = 32 * (4 + kEpiWarps + kUnpWarps);
    static constexpr uint32_t kTmemCols = 2 * BN;
    static constexpr int kColsPerWarp = BN / (kEpiWarps / 4);
    // (sc, b) per column: one private kColsPerWarp slice per epilogue warp
    // (loaded one tile ahead; no epilogue-wide barrier per tile), or (kLn)
    // (sc, b, gamma, beta) of the BN fixed columns + the quadrant partial sums
    static constexpr int kScb = kLn ? BN * 16 + (kEpiWarps / 4) * BM * 8 : kEpiWarps * kColsPerWarp * 8;
    // per epilogue warp: kLut4 one or (8 warps) two 32 x 16 B int4 blocks
    // (double-buffered TMA stores), else one 32 x 64 B output block; kLn
    // stores from registers
    static constexpr int kStgBufs = kLut4 && EPI_ <= 8 ? 2 : 1;
    // kLn: two 32 x 32 fp32 SWIZZLE_128B blocks (residual in / LN output out)
    // and two 32-row code blocks (<= 32 B per row) per warp
    static constexpr int kStagePerWarp = kLn ? LNB_ * (4096 + 1024) : (kLut4 ? 512 * kStgBufs : 2048);
    static constexpr int kStaging = kEpiWarps * kStagePerWarp;
    static constexpr int kTabBytes = kLn ? 0 : (kLut4 ? (int)rq::kSmem4Bytes : (int)rq::kSmemBytes);
    // kLut4 register split (setmaxnreg; must fit the launch allocation)
    static constexpr int kRegLaunch = ((65536 / kThreads) & ~7) > 255 ? 248 : ((65536 / kThreads) & ~7);
    static constexpr int kRegProd = 40;
    static constexpr int kRegUnp = kUnpWarps >= 8 ? (kLut4 ? 40 : 48) : 56;
    static constexpr int kRegEpi =
        ((kRegLaunch * kThreads - 128 * kRegProd - 32 * kUnpWarps * kRegUnp) / (32 * kEpiWarps)) & ~7;
    static_assert(!kRegSplit || (kRegEpi >= kRegLaunch && kRegEpi <= 256), "register split");
    static_assert(!kLn || (BN == 256 && !kLut4), "kLn: 256-column tiles");
    static_assert(kColsPerWarp % 32 == 0, "epilogue column split");
    static constexpr int kBarBytes = 8 * (2 * S8 + 2 * SP + 4 + (LN_ ? 2 * EPI_ : 0)) + 16;
    static constexpr int kSmem = 1024 + S8 * kStage8 + SP * kStageP + kTabBytes + kScb + kStaging + kBarBytes;
    static_assert(kSmem <= 232448, "shared memory budget");
    static_assert(BN == 256 || BN == 128, "BN");
    static_assert((S8 * kStage8 + SP * kStageP) % 1024 == 0, "staging must be 1024-aligned (SWIZZLE_128B)");
};

// Requant table: header fields in registers, cells in shared memory (read
// with explicit ld.shared).  Cells clamp at both ends, so y < y_lo and
// y >= y_hi need no special case: cell 0's "below" code is code_lo and the
// last cell's "above" code is code_hi.
struct Lut {
    float c0, inv_w;  // cell = floor(fma(y, inv_w, c0)), c0 = -y_lo*inv_w (rq::cell_of)
    int ncell;
    uint32_t cells;   // shared-window address of cell 0
};

__device__ __noinline__ int requant_direct(float y, int gelu, float s, int qmin, int qmax) {
    return rq::direct_code(y, gelu, s, qmin, qmax);
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// 16 requantized codes (low byte of each q[i] is the two's-complement code).
// 16 requantized codes as packed fields (int4 table: nibble 0..15; int8: byte)
__device__ __forceinline__ void lut_codes16(const Lut& L, const EpiParams& ep, const float (&y)[16], uint32_t (&q)[16]) {
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
#if defined(MKQ_ABL_NOLUT)   // ablation (diagnostics only): no table load
        const uint32_t ci = rq::cell_u(y[i], L.c0, L.inv_w, (uint32_t)L.ncell);
        const uint2 e = make_uint2(ci << 20, ci);
#elif defined(MKQ_ABL_LANELUT)   // ablation: conflict-free table addresses
        const uint32_t ci = rq::cell_u(y[i], L.c0, L.inv_w, (uint32_t)L.ncell);
        const uint2 e = lds64(L.cells + 8u * (((ci & 31u) << 5) | (threadIdx.x & 31u)));
#else
        const uint2 e = lds64(L.cells + 8u * rq::cell_u(y[i], L.c0, L.inv_w, (uint32_t)L.ncell));
#endif
        q[i] = __byte_perm(e.y, 0, y[i] >= __uint_as_float(e.x) ? 0x4441 : 0x4440);
        any |= e.y;
    }
    if (__builtin_expect(__any_sync(0xffffffffu, (any & 0x10000u) != 0), 0)) {
        const uint32_t fm = ep.mode == OUT_I4 ? 0xFu : 0xFFu;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint32_t e = lds64(L.cells + 8u * rq::cell_u(y[i], L.c0, L.inv_w, (uint32_t)L.ncell)).y;
            if (e & 0x10000u) q[i] = (uint32_t)requant_direct(y[i], ep.gelu, ep.s_out, ep.qmin, ep.qmax) & fm;
        }
    }
}

// Byte offset of 16-byte chunk c of staging row r for a row pitch P bytes
// (the TMA SWIZZLE_{128,64,32}B pattern for P = 128/64/32; none for 16).
__device__ __forceinline__ uint32_t stg_off(int r, int c, int P) {
    const int f = P == 128 ? (r & 7) : (P == 64 ? ((r >> 1) & 3) : (P == 32 ? ((r >> 2) & 1) : 0));
    return (uint32_t)(r * P + ((c ^ f) << 4));
}

// bytes per staged row: 4-byte outputs are staged and stored 16 columns at a
// time (64 B), 2-byte outputs 32 columns (64 B), int8 32 (32 B), int4 32 (16 B)
__device__ __forceinline__ int out_pitch(int mode) {
    return mode == OUT_F32 || mode == OUT_I32 ? 64 : (mode == OUT_I4 ? 16 : (mode == OUT_I8 ? 32 : 64));
}

// 16 outputs (columns cl..cl+15 of one accumulator row) -> staging row `r`,
// half `h2` of the 32-column block.
// scb holds (sc, b) per column with b = 0 without bias (fmaf(a, sc, +0) ==
// fl32(a*sc) for sc > 0, R4) and, when `fold`, sc pre-multiplied by 2^-8:
// fmaf((float)(256*sum), sc*2^-8, b) has the same exact product as
// fmaf((float)sum, sc, b) (both scalings are exact: 256*sum is an integer
// below 2^32 with >= 8 trailing zero bits, and sc*2^-8 is normal), so the
// int4 scaling shift folds away.
__device__ __forceinline__ void epi2_half(const EpiParams& ep, const Lut& L, bool use_table, bool fold, uint32_t scb,
                                          const uint32_t (&v)[16], uint8_t* stage, int r, int h2) {
    const int mode = ep.mode;
    const int P = out_pitch(mode);
    if (mode == OUT_I32) {
        int32_t acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = (int32_t)v[i] >> 8;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<int4*>(stage + stg_off(r, c, P)) =
                make_int4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
        return;
    }
    float y[16];
    if (fold) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const float4 sb = lds128f(scb + 8u * (uint32_t)i);   // (sc, b) of two columns, broadcast
            y[i] = __fmaf_rn(__int2float_rn((int32_t)v[i]), sb.x, sb.y);
            y[i + 1] = __fmaf_rn(__int2float_rn((int32_t)v[i + 1]), sb.z, sb.w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const float4 sb = lds128f(scb + 8u * (uint32_t)i);
            y[i] = __fmaf_rn(__int2float_rn((int32_t)v[i] >> 8), sb.x, sb.y);
            y[i + 1] = __fmaf_rn(__int2float_rn((int32_t)v[i + 1] >> 8), sb.z, sb.w);
        }
    }
    if (mode == OUT_I4 || mode == OUT_I8) {
        uint32_t q[16];
        if (use_table) {
            lut_codes16(L, ep, y, q);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
                q[i] = (uint32_t)quant_code(ep.gelu ? gelu_pinned(y[i]) : y[i], ep.s_out, ep.qmin, ep.qmax);
        }
        if (mode == OUT_I4) {
            if (!use_table) {   // table fields are already masked nibbles
#pragma unroll
                for (int i = 0; i < 16; ++i) q[i] &= 0xFu;
            }
            uint32_t a = 0, b = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a += q[i] * (1u << (4 * i));
                b += q[8 + i] * (1u << (4 * i));
            }
            *reinterpret_cast<uint2*>(stage + r * 16 + h2 * 8) = make_uint2(a, b);
        } else {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                w[i] = __byte_perm(__byte_perm(q[4 * i], q[4 * i + 1], 0x0040), __byte_perm(q[4 * i + 2], q[4 * i + 3], 0x0040),
                                   0x5410);
            *reinterpret_cast<uint4*>(stage + stg_off(r, h2, P)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return;
    }
    if (ep.gelu) {
#pragma unroll
        for (int i = 0; i < 16; ++i) y[i] = gelu_pinned(y[i]);
    }
    if (mode == OUT_F32) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<float4*>(stage + stg_off(r, c, P)) =
                make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
    } else {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            w[i] = mode == OUT_BF16 ? pack_bf16x2(y[2 * i], y[2 * i + 1]) : pack_f16x2(y[2 * i], y[2 * i + 1]);
        *reinterpret_cast<uint4*>(stage + stg_off(r, h2 * 2, P)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(stage + stg_off(r, h2 * 2 + 1, P)) = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

#ifdef MKQ_GTRACE
// Diagnostics build only (tools/trace_gemm.py): per-warp (tag, clock64) event
// log of CTA 0 of the 2-CTA GEMM.
__device__ unsigned long long* g_gtrace = nullptr;
constexpr int kGTraceSlots = 512;
#define GTRACE(tag)                                                                                    \
    do {                                                                                               \
        if (blockIdx.x < 2 && (threadIdx.x & 31) == 0 && g_gtrace && gt_n < kGTraceSlots) {           \
            const int gw = blockIdx.x * 24 + (threadIdx.x >> 5);                                        \
            g_gtrace[gw * kGTraceSlots * 2 + 2 * gt_n] = (tag);                                          \
            g_gtrace[gw * kGTraceSlots * 2 + 2 * gt_n + 1] = clock64();                                  \
            ++gt_n;                                                                                    \
        }                                                                                              \
    } while (0)
#else
#define GTRACE(tag) \
    do {            \
    } while (0)
#endif

// Polling policy per wait site.  Sleeping between polls (ptx::mbar_wait_sleep,
// -DMKQ_EXP_SLEEP) was measured 3% slower on FFN1 than the suspend-hint
// try_wait loop, so the default polls.
#ifdef MKQ_EXP_SLEEP
#define MKQ_WAIT_SLEEP(ns, bar, par) ptx::mbar_wait_sleep<ns>(bar, par)
#else
#define MKQ_WAIT_SLEEP(ns, bar, par) ptx::mbar_wait(bar, par)
#endif

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// A register the compiler cannot prove warp-uniform or constant: keeps values
// used by every output in one vector register (a uniform value feeding an FFMA
// that already takes a uniform operand is otherwise re-copied per use, and a
// folded constant is re-added per use).
__device__ __forceinline__ uint32_t lane_reg(uint32_t x) {
    uint32_t r;
    asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(x), "r"(threadIdx.x & 31));
    return r;
}

// a - b as an IMAD (FMA pipe; the epilogue is bound by the ALU pipe)
__device__ __forceinline__ uint32_t sub_fma(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 0xFFFFFFFF, %2;" : "=r"(r) : "r"(b), "r"(a));
    return r;
}

// 32 int4 requantized codes of one accumulator row (columns cl..cl+31) through
// the compact table (requant.cuh, "compact int4 table"): per output one cell
// computation, one conflict-free 32-bit lookup (tabm = this lane's replica
// minus the cell bias), one fp32 compare and a byte gather; outputs within the
// threshold word's direct-evaluation window (rq::kWin4), or all outputs when
// the table is unusable, are evaluated directly.  scb: (sc, sc', b, b') per
// column pair (f32x2 dequant).  Per output about 10 instructions: I2F, 1/2
// FFMA2 + 1/2 LDS.128 (dequant), FFMA.SAT + 1/2 FFMA2 + IMAD (cell address),
// LDS, IMAD + 1/2 VIMNMX3 (window), FSETP + SHF (decision), 1 PRMT/LOP3
// (nibble packing).
template <bool kFold>
__device__ __forceinline__ void epi_lut4(const EpiParams& ep, const uint32_t (&v)[32], uint32_t scb, uint32_t tabm,
                                         float a4, float b4, bool tvalid, uint32_t (&w)[4]) {
    // Two halves of 16 outputs (bounds the live registers: v[32] + y[16] + e[16]):
    // phase 1 y (dequant as f32x2), phase 2 all 16 cell addresses and table
    // loads in flight, phase 3 the decisions, the (rare, warp-uniform) direct
    // evaluation of window lanes while y is still live, the byte gather.
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const float4 sb = lds128f(scb + 8u * (uint32_t)(16 * hh + i));
            const int32_t a0 = kFold ? (int32_t)v[16 * hh + i] : ((int32_t)v[16 * hh + i] >> 8);
            const int32_t a1 = kFold ? (int32_t)v[16 * hh + i + 1] : ((int32_t)v[16 * hh + i + 1] >> 8);
            const float2 yy = fma2(make_float2(__int2float_rn(a0), __int2float_rn(a1)), make_float2(sb.x, sb.y),
                                   make_float2(sb.z, sb.w));
            y[i] = yy.x;
            y[i + 1] = yy.y;
        }
        uint32_t e[16];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const float2 cf = fma2(make_float2(rq::fma_sat(y[i], a4, b4), rq::fma_sat(y[i + 1], a4, b4)),
                                   make_float2(255.0f, 255.0f), make_float2(8388608.0f, 8388608.0f));
            e[i] = __float_as_uint(cf.x) * 128u + tabm;
            e[i + 1] = __float_as_uint(cf.y) * 128u + tabm;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
#ifdef MKQ_ABL_L4NOLUT   // ablation (diagnostics only)
            e[i] = e[i] * 0x01010101u;
#else
            e[i] = lds32(e[i]);
#endif
        }
        uint32_t bad = tvalid ? 0xFFFFFFFFu : 0u;
#pragma unroll
        for (int ii = 0; ii < 16; ++ii) {
            bad = min(bad, sub_fma(__float_as_uint(y[ii]), e[ii]));   // bits(y) - word (rq::kWin4 window)
            e[ii] = y[ii] >= __uint_as_float(e[ii]) ? (e[ii] >> 4) : e[ii];   // code in the low nibble
        }
        if (__builtin_expect(__any_sync(0xffffffffu, bad < rq::kWin4), 0)) {
            // mask of this lane's window outputs, then one call site in a loop
            // over the set bits (register selects, no local-memory indexing)
            uint32_t nm = 0;
#pragma unroll
            for (int ii = 0; ii < 16; ++ii) {
                const uint32_t ew = lds32(tabm + __float_as_uint(__fmaf_rn(rq::fma_sat(y[ii], a4, b4), 255.0f,
                                                                           8388608.0f)) * 128u);
                if (!tvalid || __float_as_uint(y[ii]) - ew < rq::kWin4) nm |= 1u << ii;
            }
            while (nm) {
                const int i = __ffs(nm) - 1;
                nm &= nm - 1;
                float yv = y[0];
#pragma unroll
                for (int k = 1; k < 16; ++k) yv = k == i ? y[k] : yv;
                const uint32_t c = (uint32_t)requant_direct(yv, ep.gelu, ep.s_out, ep.qmin, ep.qmax);
#pragma unroll
                for (int k = 0; k < 16; ++k) e[k] = k == i ? c : e[k];
            }
        }
        // nibble packing: bytes of the even / odd codes gathered with PRMT, then
        // w = (even & 0x0F0F0F0F) | ((odd << 4) & 0xF0F0F0F0) in one LOP3
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const uint32_t* f = e + 8 * g;
            const uint32_t ev = __byte_perm(__byte_perm(f[0], f[2], 0x0040), __byte_perm(f[4], f[6], 0x0040), 0x5410);
            const uint32_t od = __byte_perm(__byte_perm(f[1], f[3], 0x0040), __byte_perm(f[5], f[7], 0x0040), 0x5410);
            w[2 * hh + g] = (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
        }
    }
}

__device__ __forceinline__ void st_relaxed_gpu_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Acquire load of a global arrival counter (polled by one lane).
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Fused all-gather (NEXT(4), column-parallel FFN): the compact-table int4
// epilogue stores every output tile into `n` gathered buffers (this rank's
// and its peers', mapped into this process) at column `col0` + n, then each
// CTA signals every buffer owner's counter once (system-scope release) after
// its stores are complete.
constexpr int kMaxGather = 8;
struct GatherMaps {
    CUtensorMap m[kMaxGather];
    uint32_t* counters[kMaxGather];
    int n, col0;
};

// Tensor maps of the kLn epilogue: residual and LN output fp32 [M, N] in
// 32 x 32 SWIZZLE_128B boxes, the codes [M, N*qbits/8] in 32-row boxes of
// 16 (int4) or 32 (int8) bytes.
struct LnMaps {
    CUtensorMap r, y, q;
};

// kLn epilogue (Ln2Params): per tile, thread = one row of this CTA's 128, warp
// = one TMEM lane quadrant x kColsPerWarp columns.  The row's residual comes
// in by TMA (32 x 32 fp32 SWIZZLE_128B boxes, two per warp in flight; lane l
// reads its row's 16-byte chunks conflict-free), the accumulator is read once
// (dequant exactly as the plain epilogue: fma((float)acc, fl(s_a s_w[n])
// [2^-8 folded], b[n])), r = y + res (R9) is kept in registers and the TMEM
// buffer released.  Row statistics: each warp's (mean, M2 = sum (r - mean)^2)
// of its columns, combined over the warps of the quadrant and then over the
// np column tiles of the row group (Chan et al.'s pairwise update, fixed
// order: identical results in every CTA) through the group's `stats` slot,
// one arrival per (CTA, quadrant) on the slot's counter.  Output: y = (r -
// mean) * rstd * gamma + beta with rstd = rsqrt(M2 / N + eps) (the centred
// two-pass statistics of residual_ln), staged in the same swizzled boxes and
// TMA-stored, and optionally its Eq.1 codes.
template <class Cfg>
__device__ __forceinline__ void ln_epilogue(const Epi2Params& p, const LnMaps& lm, uint32_t tmem_base, uint64_t* tfull,
                                            uint64_t* tempty, uint64_t* rbars, uint8_t* staging, float* colp_raw,
                                            int t_begin, int t_step, int t_end, int group, int j, int M, int N,
                                            int rank) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, kCW = Cfg::kColsPerWarp, kQW = Cfg::kEpiWarps / 4;
    constexpr int kCh = kCW / 32;
    constexpr int kEpiThreads = 32 * Cfg::kEpiWarps;
    static_assert(kCh % 2 == 0, "chunk pairs");
    const EpiParams& ep = p.e;
    const Ln2Params& L = p.ln;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = warp - 4, q = warp & 3, hsl = e >> 2;   // quadrant, column slice
    const int et = threadIdx.x - 128;
    const int np = L.np;
    const int ncol0 = j * BN;                              // this pair's columns [ncol0, +BN)
    // column parameters (fixed for the whole kernel) per column pair c2:
    // dq[c2] = (sc, sc', b, b') (dequant, f32x2), ln[c2] = (g, g', beta, beta')
    float4* dq = reinterpret_cast<float4*>(colp_raw);
    float4* lnp = dq + BN / 2;
    float2* qpart = reinterpret_cast<float2*>(colp_raw + 4 * BN);   // [kQW][BM] (mean, M2) per warp slice
    float* dqf = reinterpret_cast<float*>(dq);
    float* lnf = reinterpret_cast<float*>(lnp);
    bool tiny = false;
    for (int c = et; c < BN; c += kEpiThreads) {
        const int n = ncol0 + c, o4 = 4 * (c >> 1) + (c & 1);
        const float sc = __fmul_rn(ep.s_a, __ldg(ep.s_w + n));
        tiny = tiny || !(sc >= 0x1p-118f);
        dqf[o4] = sc;
        dqf[o4 + 2] = ep.bias ? __ldg(ep.bias + n) : 0.0f;
        lnf[o4] = __ldg(L.g + n);
        lnf[o4 + 2] = __ldg(L.b + n);
    }
    const bool fold = !ptx::named_bar_sync_or(1, kEpiThreads, tiny);
    if (fold)
        for (int c = et; c < BN; c += kEpiThreads) {
            const int o4 = 4 * (c >> 1) + (c & 1);
            dqf[o4] = __fmul_rn(dqf[o4], 0x1p-8f);
        }
    ptx::named_bar_sync(1, kEpiThreads);
    const QuantRcp Qr = quant_rcp(L.s_q, L.qmin, L.qmax);
    const int row_l = q * 32 + lane;                       // row within the CTA's 128
    const int c0 = hsl * kCW;                              // first column of this warp's slice
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint8_t* stg = staging + e * Cfg::kStagePerWarp;       // [2] x 4 KB boxes, [2] x 1 KB code blocks
    const uint32_t stg_s = ptx::smem_u32(stg);
    uint64_t* rb = rbars + 2 * e;
    uint32_t rph[2] = {0u, 0u};   // per box (NB <= 2)
    // lane l's 16-byte chunk c4 of its row in a SWIZZLE_128B 32 x 128 B box
    auto sw = [lane](int c4) { return (uint32_t)(lane * 128 + ((c4 ^ (lane & 7)) << 4)); };
    uint64_t* stats_g = reinterpret_cast<uint64_t*>(L.stats) + (size_t)group * (2 * np * 2 * BM);
    const uint32_t dq_s = ptx::smem_u32(dq), ln_s = ptx::smem_u32(lnp);
    if (lane == 0) {
        ptx::tma_prefetch_desc(&lm.r);
        ptx::tma_prefetch_desc(&lm.y);
        if (L.qbits) ptx::tma_prefetch_desc(&lm.q);
    }
#ifdef MKQ_GTRACE
    int gt_n = 0;
#endif
    constexpr int NB = Cfg::kBoxes;
    auto load_res = [&](int tl, int ch) {   // TMA: residual box (tile tl, chunk ch) into box ch % NB
        if (lane == 0 && tl < t_end) {
            ptx::mbar_arrive_expect_tx(&rb[ch % NB], 4096);
            ptx::tma_load_2d(&lm.r, &rb[ch % NB], stg + (ch % NB) * 4096, ncol0 + c0 + 32 * ch,
                             tl * 2 * BM + rank * BM + q * 32);
        }
    };
    int it = 0;
    for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
        const int ab = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        const int mrow = tile * 2 * BM + rank * BM + q * 32;   // first row of this warp's 32
        GTRACE(40);
        // both boxes must have been read by the previous tile's output stores
        if (lane == 0) ptx::tma_store_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int b = 0; b < NB; ++b) load_res(tile, b);
        ptx::mbar_wait_sleep<64>(&tfull[ab], aph);
        GTRACE(42);
        ptx::tc_fence_after();
        float r[kCW];
#pragma unroll
        for (int ch = 0; ch < kCh; ++ch) {
            GTRACE(52);
            ptx::mbar_wait(&rb[ch % NB], rph[ch % NB]);
            rph[ch % NB] ^= 1u;
            GTRACE(53);
#pragma unroll
            for (int hv = 0; hv < 2; ++hv) {   // 16 accumulator columns at a time (register budget)
            uint32_t v16[16];
            ptx::tmem_ld_32x32b_x16(tmem_base + lane_off + ab * BN + c0 + 32 * ch + 16 * hv, v16);
            ptx::tmem_ld_wait();
            const uint32_t* v = v16 - 16 * hv;   // v[i] for i in [16 hv, 16 hv + 16)
#pragma unroll
            for (int c4 = 4 * hv; c4 < 4 * hv + 4; ++c4) {
                const float4 rs = lds128f(stg_s + (ch % NB) * 4096 + sw(c4));
#pragma unroll
                for (int t = 0; t < 4; t += 2) {
                    const int i = 4 * c4 + t;
                    const float4 cp = lds128f(dq_s + 16u * (uint32_t)((c0 + 32 * ch + i) >> 1));   // (sc, sc', b, b')
                    const int32_t a0 = fold ? (int32_t)v[i] : ((int32_t)v[i] >> 8);
                    const int32_t a1 = fold ? (int32_t)v[i + 1] : ((int32_t)v[i + 1] >> 8);
                    const float2 y = fma2(make_float2(__int2float_rn(a0), __int2float_rn(a1)), make_float2(cp.x, cp.y),
                                          make_float2(cp.z, cp.w));
                    const float2 rr = add2(y, t == 0 ? make_float2(rs.x, rs.y) : make_float2(rs.z, rs.w));
                    r[32 * ch + i] = rr.x;
                    r[32 * ch + i + 1] = rr.y;
                }
            }
            }
            if (ch + NB < kCh) {   // this box is consumed: refill it with chunk ch + NB
                ptx::fence_proxy_async_smem();
                __syncwarp();
                load_res(tile, ch + NB);
            }
        }
        // the accumulator buffer is free for the MMA of tile it+2
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(&tempty[ab], 0));
        GTRACE(43);
        // this warp's (mean, M2) over its kCW columns (4 f32x2 partial sums)
        float2 sp[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < kCW; i += 2) sp[(i >> 1) & 3] = add2(sp[(i >> 1) & 3], make_float2(r[i], r[i + 1]));
        const float2 s2 = add2(add2(sp[0], sp[1]), add2(sp[2], sp[3]));
        const float mw = __fadd_rn(s2.x, s2.y) / (float)kCW;   // IEEE; kCW a power of two: an exact multiply
#pragma unroll
        for (int k = 0; k < 4; ++k) sp[k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < kCW; i += 2) {
            const float2 d = add2(make_float2(r[i], r[i + 1]), make_float2(-mw, -mw));
            sp[(i >> 1) & 3] = fma2(d, d, sp[(i >> 1) & 3]);
        }
        const float2 m22 = add2(add2(sp[0], sp[1]), add2(sp[2], sp[3]));
        const float m2 = __fadd_rn(m22.x, m22.y);
        // combine: warps of the quadrant (CTA partial over BN columns), then the
        // np CTAs of the row.  The CTA partial goes out as one 64-bit word
        // (mean, M2 with its sign bit = this slot's use parity ^ 1), single-copy
        // atomic: readers poll the words of their row until all np carry the
        // current tag -- no fence, flag or counter.  M2 >= +0, so the sign bit is
        // free; the slot starts zeroed (tag 0) and its first use writes tag 1.
        qpart[hsl * BM + row_l] = make_float2(mw, m2);
        GTRACE(44);
        ptx::named_bar_sync(2 + q, 32 * kQW);
        GTRACE(45);
        uint64_t* slot = stats_g + (size_t)ab * np * (2 * BM);
        const uint32_t tag = (((uint32_t)(it >> 1)) & 1u) ^ 1u;
        if (hsl == 0) {
            float2 c = qpart[row_l];
#pragma unroll
            for (int w = 1; w < kQW; ++w) {   // equal counts kCW: pairwise update
                const float2 o = qpart[w * BM + row_l];
                const float d = __fsub_rn(o.x, c.x);
                // (w is a compile-time constant in the unrolled loop: the IEEE
                // quotients fold to constants, no dependent division chain)
                const float nw = (float)(w * kCW), nt = (float)((w + 1) * kCW);
                c.x = __fadd_rn(c.x, __fmul_rn(d, (float)kCW / nt));
                c.y = __fadd_rn(__fadd_rn(c.y, o.y), __fmul_rn(__fmul_rn(d, d), (nw * (float)kCW) / nt));
            }
            const uint64_t word = (uint64_t)__float_as_uint(c.x) | ((uint64_t)(__float_as_uint(c.y) | (tag << 31)) << 32);
            st_relaxed_gpu_u64(slot + (size_t)j * (2 * BM) + rank * BM + row_l, word);
        }
        GTRACE(46);
        float2 part[4];
        {
            const uint64_t* src = slot + rank * BM + row_l;
            uint32_t pending = (1u << np) - 1u;
            while (true) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (jj < np && (pending >> jj & 1u)) {
                        const uint64_t wv = ld_relaxed_gpu_u64(src + (size_t)jj * (2 * BM));
                        if ((uint32_t)(wv >> 63) == tag) {
                            part[jj] = make_float2(__uint_as_float((uint32_t)wv),
                                                   __uint_as_float((uint32_t)(wv >> 32) & 0x7FFFFFFFu));
                            pending &= ~(1u << jj);
                        }
                    }
                }
                if (!pending) break;
                __nanosleep(20);
            }
        }
        GTRACE(47);
        float mean = part[0].x, M2 = part[0].y;
#pragma unroll
        for (int jj = 1; jj < 4; ++jj) {   // column tiles in order: pairwise update, counts BN
            if (jj < np) {
                const float d = __fsub_rn(part[jj].x, mean);
                const float nw = (float)(jj * BN), nt = (float)((jj + 1) * BN);   // constants (unrolled)
                mean = __fadd_rn(mean, __fmul_rn(d, (float)BN / nt));
                M2 = __fadd_rn(__fadd_rn(M2, part[jj].y), __fmul_rn(__fmul_rn(d, d), (nw * (float)BN) / nt));
            }
        }
        const float rstd = rsqrtf(__fadd_rn(__fdiv_rn(M2, (float)N), L.eps));
        // output: LN(r) staged per 32-column chunk in the swizzled boxes, TMA-stored
#pragma unroll
        for (int ch = 0; ch < kCh; ++ch) {
            uint8_t* box = stg + (ch % NB) * 4096;
            uint8_t* cbx = stg + NB * 4096 + (ch % NB) * 1024;
            GTRACE(50);
            if (lane == 0) ptx::tma_store_wait_read<NB - 1>();   // the stores of chunk ch - NB have read these
            __syncwarp();
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float4 cp = lds128f(ln_s + 16u * (uint32_t)((c0 + 32 * ch + i) >> 1));   // (g, g', beta, beta')
                const float2 d = add2(make_float2(r[32 * ch + i], r[32 * ch + i + 1]), make_float2(-mean, -mean));
                const float2 oo = fma2(mul2(d, make_float2(rstd, rstd)), make_float2(cp.x, cp.y), make_float2(cp.z, cp.w));
                o[i] = oo.x;
                o[i + 1] = oo.y;
            }
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4)
                *reinterpret_cast<float4*>(box + sw(c4)) = make_float4(o[4 * c4], o[4 * c4 + 1], o[4 * c4 + 2], o[4 * c4 + 3]);
            if (L.qbits == 4) {
                uint32_t w[4];
                bool near = false;
#pragma unroll
                for (int g8 = 0; g8 < 4; ++g8) {
                    float v8[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) v8[t] = o[8 * g8 + t];
                    w[g8] = quant_nib8_fast(v8, Qr, near);
                }
                if (__builtin_expect(near, 0)) {   // a value within 2^-18 of a rounding boundary
#pragma unroll
                    for (int g8 = 0; g8 < 4; ++g8)
                        w[g8] = quant_nib8_exact(o[8 * g8], o[8 * g8 + 1], o[8 * g8 + 2], o[8 * g8 + 3], o[8 * g8 + 4],
                                                 o[8 * g8 + 5], o[8 * g8 + 6], o[8 * g8 + 7], L.s_q, L.qmin, L.qmax);
                }
                *reinterpret_cast<uint4*>(cbx + lane * 16) = make_uint4(w[0], w[1], w[2], w[3]);
            } else if (L.qbits == 8) {
                uint32_t w[8];
#pragma unroll
                for (int g4 = 0; g4 < 8; ++g4) w[g4] = quant_byte4_rcp(o[4 * g4], o[4 * g4 + 1], o[4 * g4 + 2], o[4 * g4 + 3], Qr);
                *reinterpret_cast<uint4*>(cbx + lane * 32) = make_uint4(w[0], w[1], w[2], w[3]);
                *reinterpret_cast<uint4*>(cbx + lane * 32 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                ptx::tma_store_2d(&lm.y, box, ncol0 + c0 + 32 * ch, mrow);
                if (L.qbits) ptx::tma_store_2d(&lm.q, cbx, (ncol0 + c0 + 32 * ch) * L.qbits / 8, mrow);
                ptx::tma_store_commit();
            }
            GTRACE(51);
        }
        GTRACE(48);
    }
    if (lane == 0) ptx::tma_store_wait<0>();
}

// The kernel body, shared by gemm_w4a4_2cta_kernel (plain epilogues) and
// gemm_w4a4_ln_kernel (kLn); `lm` is dereferenced only by the kLn epilogue.
template <class Cfg>
__device__ __forceinline__ void gemm2_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmO,
                                           const Epi2Params& p, int M, int N, int K, const LnMaps* lmp,
                                           const GatherMaps* gm = nullptr) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, BNH = Cfg::BNH, S8 = Cfg::S8, SP = Cfg::SP;
    constexpr int kEpiThreads = 32 * Cfg::kEpiWarps;
    constexpr int kUnpThreads = 32 * Cfg::kUnpWarps;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring8 = smem;
    uint8_t* ringP = ring8 + S8 * Cfg::kStage8;
    uint8_t* staging = ringP + SP * Cfg::kStageP;   // 1024-aligned, 4 KB per epilogue warp
    rq::Header* th = reinterpret_cast<rq::Header*>(staging + Cfg::kStaging);
    uint2* tcells = reinterpret_cast<uint2*>(th + 1);
    float2* scb = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(th) + Cfg::kTabBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(scb) + Cfg::kScb);
    uint64_t* full8 = bars;
    uint64_t* empty8 = full8 + S8;
    uint64_t* fullP = empty8 + S8;
    uint64_t* emptyP = fullP + SP;
    uint64_t* tfull = emptyP + SP;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint64_t* rbars = tempty + 4;   // kLn: [kEpiWarps][2] residual TMA barriers (after the TMEM slot)

    const EpiParams& ep = p.e;
#ifdef MKQ_GTRACE
    int gt_n = 0;
#endif
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const int cluster = blockIdx.x >> 1;
    const int nclusters = gridDim.x >> 1;
    const int m_tiles = (M + 2 * BM - 1) / (2 * BM);
    const int n_tiles = (N + BN - 1) / BN;
    const int nk = (K + Cfg::BK - 1) / Cfg::BK;
    // Tile schedule: tiles t_begin, t_begin + t_step, ... < t_end; tile -> output
    // rows [tm0(t), +256) (this CTA: + rank*128) and columns [tn0(t), +BN).
    // Default: pair `cluster` walks the (m, n) tiles.  kLn: the np pairs of a
    // group take the np column tiles of the same row tiles (pairs past the
    // last full group idle).
    int t_begin = cluster, t_step = nclusters, t_end = m_tiles * n_tiles, ln_group = 0, ln_j = 0;
    if constexpr (Cfg::kLn) {
        const int np = p.ln.np, groups = nclusters / np;
        ln_group = cluster / np;
        ln_j = cluster % np;
        t_begin = ln_group;
        t_step = groups;
        t_end = ln_group < groups ? m_tiles : 0;
    }
    auto tm0 = [&](int t) { return Cfg::kLn ? t * 2 * BM : (t / n_tiles) * 2 * BM; };
    auto tn0 = [&](int t) { return Cfg::kLn ? ln_j * BN : (t % n_tiles) * BN; };

    if (threadIdx.x == 0) {
        for (int i = 0; i < S8; ++i) {
            ptx::mbar_init(&full8[i], 2 * Cfg::kUnpWarps);   // one arrive per unpack warp of each CTA
            ptx::mbar_init(&empty8[i], 1);

        }
        for (int i = 0; i < SP; ++i) {
            ptx::mbar_init(&fullP[i], 1);
            ptx::mbar_init(&emptyP[i], kUnpThreads);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 2 * Cfg::kEpiWarps);
        }
        if constexpr (Cfg::kLn)
            for (int i = 0; i < 2 * Cfg::kEpiWarps; ++i) ptx::mbar_init(&rbars[i], 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
    }
    if (warp == 2) ptx::tmem_alloc_2cta<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    __syncthreads();   // CTA barrier as well (orders the slot write for tools that do not model barrier.cluster)
    // kLn CTAs wait on each other (row statistics): dependents are not released
    // early, so a dependent grid can never hold SMs this grid still needs
    if constexpr (!Cfg::kLn) ptx::pdl_launch();
    ptx::pdl_wait();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // kLut4: register reallocation per warpgroup (each executes one setmaxnreg
    // at one PC): producer/MMA group kRegProd, unpack kRegUnp, epilogue (the
    // latency-bound role) the rest of the launch allocation, kRegEpi
    if (warp < 4) {
    if constexpr (Cfg::kRegSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::kRegProd));
    if (warp == 0) {
        // ---------------------------------------------------- TMA producer (both CTAs)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int tile = t_begin; tile < t_end; tile += t_step) {
                const int m0 = tm0(tile) + (int)rank * BM;
                const int n0 = tn0(tile) + (int)rank * BNH;
                for (int kb = 0; kb < nk; ++kb) {
                    MKQ_WAIT_SLEEP(64, &emptyP[s], ph ^ 1);
                    uint8_t* dst = ringP + s * Cfg::kStageP;
                    ptx::mbar_arrive_expect_tx(&fullP[s], Cfg::kStageP);
                    ptx::tma_load_2d(&tmA, &fullP[s], dst, kb * (Cfg::BK / 2), m0);
                    ptx::tma_load_2d(&tmB, &fullP[s], dst + Cfg::kAP, kb * (Cfg::BK / 2), n0);
                    if (++s == SP) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------- MMA issuer (leader CTA)
        // Whole warp converged; elect.sync inside the MMA/commit wrappers picks
        // the issuing lane (3x cheaper per MMA than a diverged single lane).
        if (rank == 0) {
            constexpr uint32_t idesc = ptx::idesc_i8(2 * BM, BN);
            const uint64_t dA0 = ptx::desc_sw128_kmajor(ptx::smem_u32(ring8));
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
                const int ab = it & 1;
                const uint32_t aph = (it >> 1) & 1;
                GTRACE(29);
                MKQ_WAIT_SLEEP(32, &tempty[ab], aph ^ 1);
                GTRACE(30);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + ab * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    ptx::mbar_wait(&full8[s], ph);
                    GTRACE(31);
                    ptx::tc_fence_after();
                    const uint64_t da = dA0 + (uint64_t)((s * Cfg::kStage8) >> 4);
                    const uint64_t db = da + (uint64_t)(Cfg::kA8 >> 4);
#ifndef MKQ_ABL_NOMMA
#pragma unroll
                    for (int k = 0; k < Cfg::BK / 32; ++k)
                        ptx::mma_i8_ss_2cta_warp(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
#endif
                    ptx::mma_commit_2cta_mc_warp(&empty8[s], 3);
                    if (++s == S8) { s = 0; ph ^= 1; }
                }
                ptx::mma_commit_2cta_mc_warp(&tfull[ab], 3);
            }
        }
    }
    } else if (warp < 4 + Cfg::kEpiWarps) {
        if constexpr (Cfg::kRegSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::kRegEpi));
        // ---------------------------------------------------- epilogue (both CTAs)
        if constexpr (Cfg::kLn) {
            ln_epilogue<Cfg>(p, *lmp, tmem_base, tfull, tempty, rbars, staging, reinterpret_cast<float*>(scb), t_begin,
                             t_step, t_end, ln_group, ln_j, M, N, (int)rank);
        } else {
        const int e = warp - 4;           // 0..7
        const int q = warp & 3;           // TMEM lane quadrant (warp % 4)
        const int h = e >> 2;             // column part (kColsPerWarp columns)
        const int et = threadIdx.x - 128; // 0..255
        bool use_table = false;
        float a4 = 0.0f, b4 = 0.0f;
        if constexpr (Cfg::kLut4) {
            // replicate each compact-table word 32 times (word c*32 + l for lane l)
            const uint8_t* tg = reinterpret_cast<const uint8_t*>(p.table);
            const rq::Header* hg = reinterpret_cast<const rq::Header*>(tg);
            const rq::Header4* h4 = reinterpret_cast<const rq::Header4*>(tg + rq::kOff4);
            const uint32_t* c4 = reinterpret_cast<const uint32_t*>(h4 + 1);
            uint32_t* dst = reinterpret_cast<uint32_t*>(th);
            for (int i = et; i < rq::kCells4 * 32; i += kEpiThreads) dst[i] = __ldg(c4 + (i >> 5));
            use_table = h4->valid != 0 && hg->gelu == ep.gelu && hg->s_out == ep.s_out && hg->qmin == ep.qmin &&
                        hg->qmax == ep.qmax;
            a4 = h4->a;
            b4 = h4->b;
        } else if (p.table) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(p.table);
            uint32_t* dst = reinterpret_cast<uint32_t*>(th);
            for (int i = et; i < (int)(rq::kSmemBytes / 4); i += kEpiThreads) dst[i] = src[i];
        }
        ptx::named_bar_sync(1, kEpiThreads);
        if (!Cfg::kLut4 && p.table)
            use_table = th->valid != 0 && th->gelu == ep.gelu && th->s_out == ep.s_out && th->qmin == ep.qmin &&
                        th->qmax == ep.qmax;
        Lut L{0.0f, 0.0f, 1, ptx::smem_u32(tcells)};
        if (use_table) L = Lut{th->c0, th->inv_w, th->ncell, ptx::smem_u32(tcells)};
        uint8_t* stage = staging + e * Cfg::kStagePerWarp;
        if (lane == 0) ptx::tma_prefetch_desc(&tmO);
        // kLut4: (sc, b) of this warp's columns of the NEXT tile, loaded one tile ahead
        constexpr int kCW = Cfg::kColsPerWarp / 32;
        float2 v2[kCW];
        auto load_scales = [&](int tl) {
#pragma unroll
            for (int c = 0; c < kCW; ++c) {
                const int n = (tl % n_tiles) * BN + h * Cfg::kColsPerWarp + 32 * c + lane;
                float sw = 1.0f, bn = 0.0f;
                if (tl < t_end && n < N) {
                    sw = __ldg(ep.s_w + n);
                    bn = ep.bias ? __ldg(ep.bias + n) : 0.0f;
                }
                v2[c] = make_float2(sw, bn);
            }
        };
        load_scales(t_begin);
        // this lane's replica of the compact table, and the same minus the cell
        // bias (bits(2^23) * 128 = 2^31 mod 2^32), held in vector registers
        const uint32_t tab = ptx::smem_u32(th) + 4u * (uint32_t)lane;
        const uint32_t tabm = lane_reg(tab - (rq::kMagic << 7));
        a4 = __uint_as_float(lane_reg(__float_as_uint(a4)));
        int it = 0;
        for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
            const int m0 = tm0(tile) + (int)rank * BM;
            const int n0 = tn0(tile);
            const int ab = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            if constexpr (Cfg::kLut4) {
                // per-warp (sc, b) of this warp's kColsPerWarp columns: no epilogue-wide
                // barrier per tile, warps slip freely against each other
                float2* wsb = scb + e * Cfg::kColsPerWarp;
                bool ok = true;
#pragma unroll
                for (int c = 0; c < kCW; ++c) {
                    v2[c].x = __fmul_rn(ep.s_a, v2[c].x);   // sc = fl(s_a * s_w[n]) (R4); 1.0 * s_a past N
                    ok = ok && v2[c].x >= 0x1p-118f;
                }
                GTRACE(1);
                const bool wfold = __all_sync(0xffffffffu, ok);
                __syncwarp();
#pragma unroll
                for (int c = 0; c < Cfg::kColsPerWarp / 32; ++c)
                {   // layout per column pair: (sc_even, sc_odd, b_even, b_odd)
                    const int col = 32 * c + lane;
                    float* f = reinterpret_cast<float*>(wsb) + 4 * (col >> 1) + (col & 1);
                    f[0] = wfold ? __fmul_rn(v2[c].x, 0x1p-8f) : v2[c].x;
                    f[2] = v2[c].y;
                }
                __syncwarp();
                load_scales(tile + t_step);   // in flight during this tile
                GTRACE(2);
                // Accumulator wait.  Default: every warp sleeps between polls
                // (test_wait + nanosleep): the suspend-hint try_wait wakes on every
                // barrier event of the CTA, and sixteen epilogue warps polling with
                // it spun through ~20% of the SM's issue slots (r02 profile).
                // MKQ_EPI_ONE_POLLER: one warp polls, the rest block on a named
                // barrier (this phase-locks the warps' TMEM reads at the tile start).
#ifdef MKQ_EPI_ONE_POLLER
                if (e == 0) ptx::mbar_wait(&tfull[ab], aph);
                ptx::named_bar_sync(2, kEpiThreads);
#elif defined(MKQ_EPI_WAIT_NS)
#if MKQ_EPI_WAIT_NS == 0
                ptx::mbar_wait(&tfull[ab], aph);
#else
                ptx::mbar_wait_sleep<MKQ_EPI_WAIT_NS>(&tfull[ab], aph);
#endif
#else
                ptx::mbar_wait_sleep<64>(&tfull[ab], aph);
#endif
                GTRACE(3);
                ptx::tc_fence_after();
                const int row0 = m0 + q * 32;
                constexpr int kCh = Cfg::kColsPerWarp / 32;
                const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + ab * BN + h * Cfg::kColsPerWarp;
                // TMEM readback one chunk ahead (tcgen05.ld of chunk j+1 in flight
                // while chunk j is computed; wait::ld covers all of a thread's loads,
                // so it is issued after chunk j's work) when the registers allow it
                constexpr bool kPrefetch = Cfg::kRegEpi >= 160;
                uint32_t va[32], vb[32];
                ptx::tmem_ld_32x32b_x32(tb, va);
                ptx::tmem_ld_wait_regs(va);
                auto chunk = [&](int j, uint32_t (&cur)[32], uint32_t (&nxt)[32]) {
                    if (kPrefetch && j + 1 < kCh) ptx::tmem_ld_32x32b_x32(tb + 32 * (j + 1), nxt);
                    const int n = n0 + h * Cfg::kColsPerWarp + 32 * j;
                    GTRACE(5);
                    uint32_t w[4];
                    const uint32_t sba = ptx::smem_u32(wsb + 32 * j);
                    // unfolded tile (a column scale too small to absorb the 2^-8;
                    // rare): shift the accumulators here, so one copy of the
                    // epilogue code serves both (scb then holds the plain sc)
                    if (__builtin_expect(!wfold, 0)) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) cur[i] = (uint32_t)((int32_t)cur[i] >> 8);
                    }
                    epi_lut4<true>(ep, cur, sba, tabm, a4, b4, use_table, w);
                    GTRACE(6);
                    // staging block(s): the store that last used this block must
                    // have read it
                    uint8_t* stg = stage + 512 * (j % Cfg::kStgBufs);
                    if (lane == 0) ptx::tma_store_wait_read<Cfg::kStgBufs - 1>();
                    __syncwarp();
                    *reinterpret_cast<uint4*>(stg + lane * 16) = make_uint4(w[0], w[1], w[2], w[3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
#ifndef MKQ_ABL_L4NOSTORE
                    if (lane == 0 && n < N) {
                        if (gm) {   // fused all-gather: the tile into every rank's gathered buffer
                            for (int g = 0; g < gm->n; ++g) ptx::tma_store_2d(&gm->m[g], stg, (gm->col0 + n) / 2, row0);
                        } else {
                            ptx::tma_store_2d(&tmO, stg, n / 2, row0);
                        }
                        ptx::tma_store_commit();
                    }
#endif
                    if (j + 1 < kCh) {
                        if (!kPrefetch) ptx::tmem_ld_32x32b_x32(tb + 32 * (j + 1), nxt);
                        ptx::tmem_ld_wait_regs(nxt);
                    }
                };
                static_assert(kCh % 2 == 0, "chunk pairs");
#ifndef MKQ_ABL_NOEPI
#pragma unroll 1
                for (int j = 0; j < kCh; j += 2) {
                    chunk(j, va, vb);
                    chunk(j + 1, vb, va);
                }
#endif
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(&tempty[ab], 0));
                GTRACE(8);
                continue;
            }
            // per-warp (sc, b) of this warp's kColsPerWarp columns (loaded one tile
            // ahead), written as one float2 per column; the 2^-8 fold is decided per
            // warp (folded and unfolded dequant give identical bits, R4)
            float2* wsb = scb + e * Cfg::kColsPerWarp;
            bool ok = true;
#pragma unroll
            for (int c = 0; c < kCW; ++c) {
                v2[c].x = __fmul_rn(ep.s_a, v2[c].x);   // sc = fl(s_a * s_w[n]) (R4); 1.0 * s_a past N
                ok = ok && v2[c].x >= 0x1p-118f;
            }
            const bool fold = __all_sync(0xffffffffu, ok);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < kCW; ++c)
                wsb[32 * c + lane] = make_float2(fold ? __fmul_rn(v2[c].x, 0x1p-8f) : v2[c].x, v2[c].y);
            __syncwarp();
            load_scales(tile + t_step);   // in flight during this tile
            ptx::mbar_wait_sleep<64>(&tfull[ab], aph);
            ptx::tc_fence_after();
            const int row0 = m0 + q * 32;
            {
#pragma unroll 1
            for (int j = 0; j < Cfg::kColsPerWarp / 32; ++j) {
                const int cl = h * Cfg::kColsPerWarp + 32 * j;
                const int n = n0 + cl;
                if (n >= N) break;
                const bool wide = ep.mode == OUT_F32 || ep.mode == OUT_I32;   // two 16-column stores
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    if (h2 == 0 || wide) {
                        // the previous TMA store must have finished reading the staging block
                        if (lane == 0) ptx::tma_store_wait_read<0>();
                        __syncwarp();
                    }
                    uint32_t v[16];
                    ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(q * 32) << 16) + ab * BN + cl + 16 * h2, v);
                    ptx::tmem_ld_wait();
                    epi2_half(ep, L, use_table, fold, ptx::smem_u32(wsb + (cl - h * Cfg::kColsPerWarp) + 16 * h2), v,
                              stage, lane, h2);
                    if (h2 == 1 || wide) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
#ifndef MKQ_ABL_NOSTORE2   // ablation (diagnostics only): no output store
                        if (lane == 0) {
                            const int nn = n + (wide ? 16 * h2 : 0);
                            ptx::tma_store_2d(&tmO, stage, ep.mode == OUT_I4 ? nn / 2 : nn, row0);
                            ptx::tma_store_commit();
                        }
#endif
                    }
                }
            }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(&tempty[ab], 0));
        }
        if (lane == 0) ptx::tma_store_wait<0>();
        if (gm) {
            // this warp's stores are complete; make them visible beyond the GPU, then
            // one release increment per CTA on every gathered buffer's owner counter
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence_system();
            }
            __syncwarp();
            ptx::named_bar_sync(1, kEpiThreads);
            if (threadIdx.x == 128)
                for (int g = 0; g < gm->n; ++g)
                    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(gm->counters[g]) : "memory");
        }
        }
    } else {
        if constexpr (Cfg::kRegSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::kRegUnp));
        // ---------------------------------------------------- int4 -> int8 unpack (both CTAs)
        const int u = threadIdx.x - 32 * (4 + Cfg::kEpiWarps);
        constexpr int kChunks = (BM + BNH) * (Cfg::BK / 32);   // 16-byte packed chunks per stage
        constexpr int kPer = kChunks / kUnpThreads;
        static_assert(kChunks % kUnpThreads == 0, "chunk split");
        constexpr uint32_t kRowsPerPass = kUnpThreads / 4;
        // Thread u always handles 16-byte chunk c = u & 3 of rows r = (u >> 2) + (threads/4) i:
        // its swizzle phase (r & 7) and both destination offsets are loop invariants.
        const uint32_t r0 = (uint32_t)u >> 2, c = (uint32_t)u & 3u, r7 = r0 & 7u;
        const uint32_t src_off = r0 * 64u + c * 16u;
        const uint32_t dlo_off = r0 * 128u + (((2u * c) ^ r7) << 4);
        const uint32_t dhi_off = r0 * 128u + (((2u * c + 1u) ^ r7) << 4);
        const uint32_t ringP_s = ptx::smem_u32(ringP), ring8_s = ptx::smem_u32(ring8);
        int sp = 0, s8 = 0;
        uint32_t php = 0, ph8 = 0;
        for (int tile = t_begin; tile < t_end; tile += t_step) {
            for (int kb = 0; kb < nk; ++kb) {
                GTRACE(19);
                MKQ_WAIT_SLEEP(32, &fullP[sp], php);
                GTRACE(20);
                const uint32_t src = ringP_s + (uint32_t)sp * Cfg::kStageP + src_off;
                uint4 pk[kPer];
#ifndef MKQ_DBG_NO_UNPACK
#pragma unroll
                for (int i = 0; i < kPer; ++i) pk[i] = ptx::lds128(src + (uint32_t)i * (kRowsPerPass * 64u));
#endif
                MKQ_WAIT_SLEEP(32, &empty8[s8], ph8 ^ 1);
                GTRACE(21);
                const uint32_t dst = ring8_s + (uint32_t)s8 * Cfg::kStage8;
#ifndef MKQ_DBG_NO_UNPACK
#pragma unroll
                for (int i = 0; i < kPer; ++i) {
                    const uint4 pv = pk[i];
                    uint4 lo, hi;
                    ptx::unpack_i4x8(pv.x, lo.x, hi.x);
                    ptx::unpack_i4x8(pv.y, lo.y, hi.y);
                    ptx::unpack_i4x8(pv.z, lo.z, hi.z);
                    ptx::unpack_i4x8(pv.w, lo.w, hi.w);
                    const uint32_t rb = dst + (uint32_t)i * (kRowsPerPass * 128u);
                    ptx::sts128(rb + dlo_off, lo);
                    ptx::sts128(rb + dhi_off, hi);
                }
#else
                (void)src; (void)dst; (void)pk;
#endif
                // release the packed stage only after its data has been consumed
                // (the STS above depend on the loaded registers): a generic-proxy
                // release does not order pending LDS against the async-proxy TMA
                // refill of the same bytes.
                ptx::mbar_arrive(&emptyP[sp]);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(&full8[s8], 0));
                if (++sp == SP) { sp = 0; php ^= 1; }
                if (++s8 == S8) { s8 = 0; ph8 ^= 1; }
            }
        }
        // tail: wait until the MMA's last multicast commits on empty8 have landed
        for (int i = 0; i < S8; ++i) {
            ptx::mbar_wait(&empty8[s8], ph8 ^ 1);
            if (++s8 == S8) { s8 = 0; ph8 ^= 1; }
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2cta<Cfg::kTmemCols>(tmem_base);
    }
}

template <class Cfg>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg::kThreads, 1)
    gemm_w4a4_2cta_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmO, const Epi2Params p, int M, int N, int K) {
    static_assert(!Cfg::kLn, "kLn: gemm_w4a4_ln_kernel");
    gemm2_body<Cfg>(tmA, tmB, tmO, p, M, N, K, nullptr);
}

template <class Cfg>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg::kThreads, 1)
    gemm_w4a4_ln_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const Epi2Params p, int M, int N, int K, const __grid_constant__ LnMaps lm) {
    static_assert(Cfg::kLn, "plain epilogues: gemm_w4a4_2cta_kernel");
    gemm2_body<Cfg>(tmA, tmB, tmA, p, M, N, K, &lm);
}

template <class Cfg>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg::kThreads, 1)
    gemm_w4a4_gather_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const Epi2Params p, int M, int N, int K, const __grid_constant__ GatherMaps gm) {
    static_assert(Cfg::kLut4, "the fused all-gather is the compact-table int4 epilogue");
    gemm2_body<Cfg>(tmA, tmB, gm.m[0], p, M, N, K, nullptr, &gm);
}

// Consumer side of the fused all-gather: block the stream until `counter`
// (this rank's, incremented by the producers' CTAs) reaches `target`.
__global__ void wait_counter_kernel(const uint32_t* counter, uint32_t target) {
    uint32_t v;
    do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if (v < target) __nanosleep(256);
    } while (v < target);
}

}  // namespace mkq

#ifdef MKQ_GTRACE
extern "C" __attribute__((visibility("default"))) int mkq_debug_set_gtrace(void* p) {
    unsigned long long* q = static_cast<unsigned long long*>(p);
    return (int)cudaMemcpyToSymbol(mkq::g_gtrace, &q, sizeof(q));
}
#endif
