// attention_pp_sm100.cuh -- §8(a) row a8 glue: the attention core of Eq.3-5
// (q k^T per R8; fp16 operands R10; fp32 softmax P:234; fused Eq.1
// quantize of OA), "ping-pong" variant for B200.
//
// One persistent CTA per SM walks work items (sequence, head, pair of
// 128-query tiles A and B).  K/V blocks of 128 keys are loaded once per pair
// (TMA, SWIZZLE_128B, 3-stage ring) and shared by both tiles.  The MMA warp
// interleaves the two tiles so the tensor core works on one while the other
// tile's softmax runs:
//     S_A(0) S_B(0) | S_A(j+1) PV_A(j) | S_B(j+1) PV_B(j) | ...
// S_X = Q_X K_j^T (tcgen05.mma kind::f16, M=128, N=128, fp32 in TMEM);
// PV_X: O_X += P_X V_j with P_X read back from TMEM (TS MMA) and V_j as an
// MN-major smem operand.  When softmax X hands over P_X(j), the MMA warp
// issues S_X(j+1) first and then PV_X(j), so the next scores are ready as
// early as possible; pv_done tells softmax X when P_X may be overwritten and
// O_X rescaled.  Softmax: 4 warps per tile, thread = query row, the
// whole 128-key row in registers (no cross-warp exchange); O accumulates in
// TMEM with lazy rescaling (reference max raised only when a block max exceeds
// it by > 2^8, so P <= 256 in fp16).
// TMEM: S_A [0,128), S_B [128,256), O_A [256,320), O_B [320,384), P_A
// [384,448), P_B [448,512) (alloc 512; P apart from S so S_X(j+1) never
// overwrites the operand PV_X(j) reads).  Q is double-buffered per item.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include "attention_sm100.cuh"
#include "epilogue.cuh"
#include "ptx.cuh"

namespace mkq {
namespace attnpp {

using attn2::desc_sw128_mnmajor;
using attn2::ex2f;
using attn2::h2;
using attn2::idesc_f16;
using attn2::mma_f16_ss;
using attn2::mma_f16_ts;
using attn2::mma_f16_ss_warp;
using attn2::mma_f16_ts_warp;
using attn2::Params;
using attn2::tmem_st_x16;
using attn2::ffma2;
using attn2::fadd2;
using attn2::ex2_fma2;
#ifndef MKQ_ATTN_POLY_FROM
#define MKQ_ATTN_POLY_FROM 6   // pairs (i & 7) >= this use the FMA-pipe exp2 (tools/attn_poly.sh: 8 537 us, 6 523, 5 549, 4 561)
#endif
constexpr int kPolyFrom = MKQ_ATTN_POLY_FROM;

constexpr int kBQ = 128, kBK = 128, kD = 64;
constexpr int kStages = 3;
constexpr int kQBytes = kBQ * kD * 2;      // 16 KB
constexpr int kKVBytes = kBK * kD * 2;     // 16 KB
// warpgroup 0: w0 TMA + TMEM alloc, w1 MMA, w2-3 idle; warpgroup 1: softmax A;
// warpgroup 2: softmax B (setmaxnreg: 56 registers for warpgroup 0, 224 for the
// softmax warpgroups, which keep a 128-score row in registers)
constexpr int kThreads = 32 * 12;
constexpr int kRegLaunch = 168, kRegCtl = 56, kRegSoft = 224;
static_assert(kRegCtl * 128 + kRegSoft * 256 <= kRegLaunch * kThreads, "register split");
constexpr float kRescale = 8.0f;
constexpr int kSmem = 1024 + 4 * kQBytes + 2 * kStages * kKVBytes + 512;

#ifdef MKQ_TRACE
// Diagnostics build only (tools/trace_attn.py): per-warp (tag, clock64)
// event log of CTA 0.
__device__ unsigned long long* g_trace = nullptr;
constexpr int kTraceSlots = 512;
#define TRACE(tag)                                                                              \
    do {                                                                                        \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && g_trace && tr_n < kTraceSlots) {      \
            g_trace[(threadIdx.x >> 5) * kTraceSlots * 2 + 2 * tr_n] = (tag);                   \
            g_trace[(threadIdx.x >> 5) * kTraceSlots * 2 + 2 * tr_n + 1] = clock64();           \
            ++tr_n;                                                                             \
        }                                                                                       \
    } while (0)
#else
#define TRACE(tag) \
    do {           \
    } while (0)
#endif

struct Item {
    int start, len, head, q0, nblk;
    bool hasB;
};

__device__ __forceinline__ bool get_item(const Params& p, int w, int heads, int pairs, Item& it) {
    const int pr = w % pairs;
    const int bh = w / pairs;
    const int h = bh % heads, b = bh / heads;
    it.start = p.cu ? p.cu[b] : b * p.seq;
    it.len = p.cu ? (p.cu[b + 1] - it.start) : p.seq;
    it.head = h;
    it.q0 = pr * 2 * kBQ;
    it.nblk = (it.len + kBK - 1) / kBK;
    it.hasB = it.q0 + kBQ < it.len;
    return it.q0 < it.len;
}

template <int kOut>   // output mode: 0 f32, 3 int4, 4 int8
__global__ void __launch_bounds__(kThreads, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const Params p, int heads, int pairs, int nitems) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                             // [buffer][tile A, B]
    uint8_t* sK = sQ + 4 * kQBytes;
    uint8_t* sV = sK + kStages * kKVBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * kKVBytes);
    uint64_t* q_full = bars;                        // [2] (both tiles)
    uint64_t* q_empty = q_full + 2;                 // [2]
    uint64_t* kv_full = q_empty + 2;                // [kStages] K_j and V_j landed
    uint64_t* pv_done = kv_full + kStages;          // [2] per tile: PV_x(j) complete (P_x reusable)
    uint64_t* kv_empty = pv_done + 2;               // [kStages]
    uint64_t* s_full = kv_empty + kStages;          // [2] per tile
    uint64_t* p_ready = s_full + 2;                 // [2] per tile
    uint64_t* o_done = p_ready + 2;                 // [2] per tile, once per item
    uint64_t* s_free = o_done + 2;                  // [2] per tile: S_x(j) read into registers (j < nblk-1)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef MKQ_TRACE
    int tr_n = 0;
#endif
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&q_full[i], 1);
            ptx::mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&kv_full[i], 1);
            ptx::mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&p_ready[i], 4);
            ptx::mbar_init(&o_done[i], 1);
            ptx::mbar_init(&pv_done[i], 1);
            ptx::mbar_init(&s_free[i], 4);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::pdl_launch();
    ptx::pdl_wait();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // S_x = tmem + x*kBK, O_x = tmem + 2*kBK + x*kD, P_x = tmem + 2*kBK + (2+x)*kD
    auto tS = [tmem](int x) { return tmem + (uint32_t)(x * kBK); };
    auto tO = [tmem](int x) { return tmem + (uint32_t)(2 * kBK + x * kD); };
    auto tP = [tmem](int x) { return tmem + (uint32_t)(2 * kBK + (2 + x) * kD); };

    // setmaxnreg inside each role's branch (ptxas then allocates each region
    // with its own budget)
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    if (warp == 0) {
        // ---------------------------------------------------- TMA producer
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmQ);
            ptx::tma_prefetch_desc(&tmKV);
            int g = 0, it = 0;
            Item I;
            for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
                if (!get_item(p, w, heads, pairs, I)) continue;
                const int colq = I.head * kD, colk = p.hidden + I.head * kD, colv = 2 * p.hidden + I.head * kD;
                const int qb = it & 1;
                ptx::mbar_wait(&q_empty[qb], ((it >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&q_full[qb], 2 * kQBytes);
                uint8_t* q_dst = sQ + qb * 2 * kQBytes;
                ptx::tma_load_2d(&tmQ, &q_full[qb], q_dst, colq, I.start + I.q0);
                ptx::tma_load_2d(&tmQ, &q_full[qb], q_dst + kQBytes, colq, I.start + I.q0 + kBQ);   // unused if !hasB
                for (int j = 0; j < I.nblk; ++j, ++g) {
                    const int st = g % kStages;
                    TRACE(40);
                    ptx::mbar_wait(&kv_empty[st], ((g / kStages) & 1) ^ 1);
                    TRACE(41);
                    ptx::mbar_arrive_expect_tx(&kv_full[st], 2 * kKVBytes);
                    ptx::tma_load_2d(&tmKV, &kv_full[st], sK + st * kKVBytes, colk, I.start + j * kBK);
                    ptx::tma_load_2d(&tmKV, &kv_full[st], sV + st * kKVBytes, colv, I.start + j * kBK);
                }
                ++it;
            }
            for (int i = 0; i < kStages; ++i, ++g) ptx::mbar_wait(&kv_empty[g % kStages], ((g / kStages) & 1) ^ 1);
            for (int i = 0; i < 2; ++i, ++it) ptx::mbar_wait(&q_empty[it & 1], ((it >> 1) & 1) ^ 1);
        }
    } else if (warp == 1) {
        // ---------------------------------------------------- MMA issuer
        // The whole warp runs this loop converged; elect.sync inside the MMA
        // and commit wrappers picks the issuing lane.  Descriptors are
        // precomputed and advanced by constants (start address field >> 4).
        constexpr uint32_t idS = idesc_f16(kBQ, kBK, 0);
        constexpr uint32_t idO = idesc_f16(kBQ, kD, 1);
        const uint64_t dQ0 = ptx::desc_sw128_kmajor(ptx::smem_u32(sQ));
        const uint64_t dK0 = ptx::desc_sw128_kmajor(ptx::smem_u32(sK));
        const uint64_t dV0 = desc_sw128_mnmajor(ptx::smem_u32(sV));
        int g = 0, it = 0, qb = 0;
        uint32_t sph[2] = {0, 0};   // number of P hand-overs per tile (p_ready parity source)
        uint32_t fph[2] = {0, 0};   // number of S read-backs per tile (s_free parity source)
        Item I;
        auto issue_S = [&](int x, int gg) {
            const uint64_t dq = dQ0 + (uint64_t)((2 * qb + x) * (kQBytes >> 4));
            const uint64_t dk = dK0 + (uint64_t)((gg % kStages) * (kKVBytes >> 4));
#pragma unroll
            for (int k = 0; k < kD / 16; ++k) mma_f16_ss_warp(tS(x), dq + 2 * k, dk + 2 * k, idS, k != 0);
            ptx::mma_commit_warp(&s_full[x]);
        };
        auto issue_PV = [&](int x, int gg, int j) {
            const uint64_t dv = dV0 + (uint64_t)((gg % kStages) * (kKVBytes >> 4));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) mma_f16_ts_warp(tO(x), tP(x) + 8 * k, dv + 128 * k, idO, (j | k) != 0);
        };
        // Per block j and tile x: as soon as softmax x hands over P_x(j)
        // (p_ready), S_x(j+1) is issued first (S_x's columns are free: P
        // lives apart), then PV_x(j); softmax x waits pv_done before it
        // overwrites P_x or rescales O_x.
        for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
            if (!get_item(p, w, heads, pairs, I)) continue;
            qb = it & 1;
            ptx::mbar_wait(&q_full[qb], (it >> 1) & 1);
            ptx::mbar_wait(&kv_full[g % kStages], (g / kStages) & 1);
            ptx::tc_fence_after();
            issue_S(0, g);
            if (I.hasB) issue_S(1, g);
            for (int j = 0; j < I.nblk; ++j, ++g) {
                const int st = g % kStages;
                const bool more = j + 1 < I.nblk;
                if (more) ptx::mbar_wait(&kv_full[(g + 1) % kStages], ((g + 1) / kStages) & 1);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    if (x == 1 && !I.hasB) break;
                    // S_x(j+1) as soon as softmax x holds S_x(j) in registers, so it
                    // computes under softmax x's exponentials (was: after P_x(j))
                    if (more) {
                        ptx::mbar_wait(&s_free[x], fph[x] & 1);
                        ++fph[x];
                        ptx::tc_fence_after();
                        issue_S(x, g + 1);
                    }
                    TRACE(10 + 10 * x);
                    ptx::mbar_wait(&p_ready[x], sph[x] & 1);
                    TRACE(11 + 10 * x);
                    ++sph[x];
                    ptx::tc_fence_after();
#ifndef MKQ_ABL_NOPV
                    issue_PV(x, g, j);
#endif
                    ptx::mma_commit_warp(&pv_done[x]);
                    if (!more) ptx::mma_commit_warp(&o_done[x]);
                    TRACE(12 + 10 * x);
                }
                ptx::mma_commit_warp(&kv_empty[st]);
            }
            ptx::mma_commit_warp(&q_empty[qb]);
            ++it;
        }
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoft));
        // ---------------------------------------------------- softmax + epilogue
        const int x = warp >= 8 ? 1 : 0;          // tile
        const int q = warp & 3;                   // TMEM lane quadrant
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float c = 0.125f * 1.4426950408889634f;   // 1/sqrt(64) * log2(e)
        uint32_t sph = 0, oph = 0;
        uint32_t nb = 0;   // blocks this tile has handed to the MMA warp (pv_done phases issued)
        Item I;
        for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
            if (!get_item(p, w, heads, pairs, I)) continue;
            if (x == 1 && !I.hasB) continue;
            TRACE(12);
            const int row = I.q0 + x * kBQ + q * 32 + lane;   // query row within the sequence
            float m = -INFINITY, l = 0.0f;
            for (int j = 0; j < I.nblk; ++j) {
                TRACE(1);
                ptx::mbar_wait(&s_full[x], sph & 1);
                TRACE(2);
                ++sph;
                ptx::tc_fence_after();
                uint32_t sv[4][32];
#pragma unroll
#ifdef MKQ_ABL_NOLD   // ablation (diagnostics only): no S readback
                for (int cc = 0; cc < 4; ++cc)
                    for (int i = 0; i < 32; ++i) sv[cc][i] = __float_as_uint((float)((lane * 7 + i * 3 + cc) & 15));
#else
                // 32 columns per load (a 4 KB x32 load costs a warp ~94 cycles with
                // or without others in flight: profiles/r02_microbench.md)
                for (int cc = 0; cc < 4; ++cc) {
                    ptx::tmem_ld_32x32b_x32(tS(x) + lane_off + 32 * cc, sv[cc]);
                    ptx::tmem_ld_wait_regs(sv[cc]);
                }
#endif
                if (j + 1 < I.nblk) {   // S_x's columns are free for S_x(j+1)
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&s_free[x]);
                }
                const int kvalid = I.len - j * kBK;   // keys >= kvalid are masked (last block only)
                if (kvalid < kBK) {
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (32 * cc + i >= kvalid) sv[cc][i] = __float_as_uint(-INFINITY);
                }
                float pm[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) pm[t] = -INFINITY;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                    for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], __uint_as_float(sv[cc][i]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) * c;
                const bool up = mx > m + kRescale;
                if (__any_sync(0xffffffffu, up)) {
                    const float m_new = up ? mx : m;
                    const float alpha = ex2f(m - m_new);   // 0 when m = -inf, 1 when !up
                    l *= alpha;
                    if (j > 0) {   // O_x must hold PV_x(j-1): wait for it
                        ptx::mbar_wait(&pv_done[x], (nb - 1) & 1);
                        ptx::tc_fence_after();
#pragma unroll
                        for (int hh = 0; hh < 4; ++hh) {   // 16 columns at a time (register pressure)
                            uint32_t o[16];
                            ptx::tmem_ld_32x32b_x16(tO(x) + lane_off + 16 * hh, o);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                            tmem_st_x16(tO(x) + lane_off + 16 * hh, o);
                        }
                    }
                    m = m_new;
                }
                // Optional (MKQ_ATTN_STAGGER, off): XU turn-taking between the two
                // tiles' warps of one quadrant (same SMSP), A(j) -> B(j) -> A(j+1).
                // Since S_x(j+1) is issued as soon as S_x(j) is read back, the
                // turn-taking only delays the tiles (535 vs 482 us at C4).
                TRACE(3);
#ifdef MKQ_ATTN_STAGGER
                if (I.hasB) {
                    if (x == 0 && j > 0) ptx::named_bar_sync(5 + q, 64);
                    if (x == 1) ptx::named_bar_sync(1 + q, 64);
                }
#endif
                TRACE(4);
                const float nmx = -m;
                float2 ps2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
                if (nb > 0) {   // P_x is free once PV_x of the previous block completed
                    ptx::mbar_wait(&pv_done[x], (nb - 1) & 1);
                    ptx::tc_fence_after();
                }
                TRACE(13);
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 x2 = ffma2(make_float2(__uint_as_float(sv[cc][2 * i]), __uint_as_float(sv[cc][2 * i + 1])),
                                                make_float2(c, c), make_float2(nmx, nmx));
#ifdef MKQ_ABL_NOEXP   // ablation (diagnostics only): no MUFU
                        const float2 e2 = x2;
#else
                        // 2 of every 8 pairs on the FMA pipe (ex2_fma2), the rest on
                        // MUFU: balances the two pipes (XU 8 cycles / FMA ~6 per element)
                        const float2 e2 = (i & 7) >= kPolyFrom ? ex2_fma2(x2) : make_float2(ex2f(x2.x), ex2f(x2.y));
#endif
                        ps2[i & 1] = fadd2(ps2[i & 1], e2);
                        pk[i] = h2(e2.x, e2.y);
                    }
#ifdef MKQ_ABL_NOST
                    if (pk[0] == 0x12345678u && pk[15] == 0x9abcdef0u)
#endif
                    tmem_st_x16(tP(x) + lane_off + 16 * cc, pk);
                }
#ifdef MKQ_ATTN_STAGGER
                if (I.hasB) {
                    if (x == 0) ptx::named_bar_arrive(1 + q, 64);
                    if (x == 1 && j + 1 < I.nblk) ptx::named_bar_arrive(5 + q, 64);
                }
#endif
                l += (ps2[0].x + ps2[1].x) + (ps2[0].y + ps2[1].y);
                TRACE(14);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&p_ready[x]);
                ++nb;
                TRACE(5);
            }
            // ---- epilogue: O / l -> quantize -> global
            TRACE(6);
            ptx::mbar_wait(&o_done[x], oph & 1);
            TRACE(7);
            ++oph;
            ptx::tc_fence_after();
            uint32_t o[2][32];
            ptx::tmem_ld_32x32b_x32(tO(x) + lane_off, o[0]);
            ptx::tmem_ld_wait_regs(o[0]);
            ptx::tmem_ld_32x32b_x32(tO(x) + lane_off + 32, o[1]);
            ptx::tmem_ld_wait_regs(o[1]);
            ptx::tc_fence_before();
            TRACE(8);
            if (row < I.len) {
                const float inv = 1.0f / l;
                uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)(I.start + row) * p.ldo;
                if constexpr (kOut == 0) {
                    float4* dst = reinterpret_cast<float4*>(orow + (int64_t)I.head * kD * 4);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int hh = i >> 3, b0 = 4 * (i & 7);
                        dst[i] = make_float4(__uint_as_float(o[hh][b0]) * inv, __uint_as_float(o[hh][b0 + 1]) * inv,
                                             __uint_as_float(o[hh][b0 + 2]) * inv, __uint_as_float(o[hh][b0 + 3]) * inv);
                    }
                } else if constexpr (kOut == 3) {
                    const QuantRcp Q = quant_rcp(p.s_out, p.qmin, p.qmax);
                    uint32_t wq[8];
#pragma unroll
                    for (int gq = 0; gq < 8; ++gq) {
                        float v[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(o[gq >> 2][8 * (gq & 3) + i]) * inv;
                        bool near = false;
                        wq[gq] = quant_nib8_fast(v, Q, near);
                        if (__builtin_expect(near, 0))   // within 2^-18 of a rounding boundary: exact Eq.1
                            wq[gq] = quant_nib8_exact(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], p.s_out, p.qmin,
                                                      p.qmax);
                    }
                    TRACE(9);
                    uint4* dst = reinterpret_cast<uint4*>(orow + I.head * kD / 2);
                    dst[0] = make_uint4(wq[0], wq[1], wq[2], wq[3]);
                    dst[1] = make_uint4(wq[4], wq[5], wq[6], wq[7]);
                } else {
                    const QuantRcp Q = quant_rcp(p.s_out, p.qmin, p.qmax);
                    uint32_t wq[16];
#pragma unroll
                    for (int gq = 0; gq < 16; ++gq) {
                        const int hh = gq >> 3, b0 = 4 * (gq & 7);
                        wq[gq] = quant_byte4_rcp(__uint_as_float(o[hh][b0]) * inv, __uint_as_float(o[hh][b0 + 1]) * inv,
                                                 __uint_as_float(o[hh][b0 + 2]) * inv,
                                                 __uint_as_float(o[hh][b0 + 3]) * inv, Q);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(orow + I.head * kD);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(wq[4 * i], wq[4 * i + 1], wq[4 * i + 2], wq[4 * i + 3]);
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

}  // namespace attnpp
}  // namespace mkq

#ifdef MKQ_TRACE
extern "C" __attribute__((visibility("default"))) int mkq_debug_set_trace(void* p) {
    unsigned long long* q = static_cast<unsigned long long*>(p);
    return (int)cudaMemcpyToSymbol(mkq::attnpp::g_trace, &q, sizeof(q));
}
#endif
