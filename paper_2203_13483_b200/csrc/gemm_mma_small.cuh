// gemm_mma_small.cuh -- latency-first W4A4 / W8A8 GEMM for small M (the
// paper's Table 2 regime), §8(a) rows a2-a7.
//
// At a few hundred rows the tcgen05 kernels are bound by their fixed
// latencies (TMEM allocation, barrier setup, TMA descriptor fetch, a staged
// epilogue), not by tensor throughput.  This kernel uses the register-level
// mma.sync IMMA path instead: 64 x 64 output tiles, 4 warps (2 x 2, each
// 32 x 32), packed tiles streamed global -> shared with cp.async through a
// 6-stage ring, int4 codes expanded in registers right before the MMA, and
// the epilogue applied to the accumulator fragments directly.
//
// int4 expansion (exact, as in gemm_sm100.cuh): a packed 32-bit word holds
// codes k..k+7; lo = (p << 4) & 0xF0F0F0F0 holds 16 x the even codes, hi =
// p & 0xF0F0F0F0 16 x the odd codes.  Thread t of an m16n8k32 fragment takes
// the word of codes [8t, 8t+8) of its row: lo as a0/a1 (fragment k = 4t..4t+3)
// and hi as a2/a3 (k = 16+4t..), and the B fragment is built the same way, so
// A and B see the same permutation of k and the s32 accumulator is exactly
// 256 * sum(a w) (|acc| <= 256 * 64 * K < 2^31 for K <= MKQ_MAX_K).
#pragma once
#include <cstdint>
#include "epilogue.cuh"
#include "gemm_sm100.cuh"

namespace mkq {
namespace gsm {

constexpr int BM = 64, BN = 64, BK = 128;   // BK in codes per stage
constexpr int kStages = 6;
constexpr int kThreads = 128;

template <bool kInt4>
struct Cfg {
    static constexpr int kRowBytes = kInt4 ? BK / 2 : BK;   // bytes per tile row per stage
    static constexpr int kPitch = kRowBytes + 16;             // padded smem pitch (conflict-free fragments)
    static constexpr int kStage = (BM + BN) * kPitch;
    static constexpr int kSmem = kStages * kStage;
};

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

__device__ __forceinline__ void imma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Two adjacent output columns (n, n+1) of one row: dequant (R4), GELU, encode.
__device__ __forceinline__ void emit2(const EpiParams& ep, int row, int n, int32_t a0, int32_t a1) {
    uint8_t* orow = reinterpret_cast<uint8_t*>(ep.out) + (int64_t)row * ep.ldo_bytes;
    if (ep.mode == OUT_I32) {
        *reinterpret_cast<int2*>(orow + (int64_t)n * 4) = make_int2(a0, a1);
        return;
    }
    const bool hb = ep.bias != nullptr;
    float y0 = dequant(a0, __fmul_rn(ep.s_a, __ldg(ep.s_w + n)), hb ? __ldg(ep.bias + n) : 0.0f, hb);
    float y1 = dequant(a1, __fmul_rn(ep.s_a, __ldg(ep.s_w + n + 1)), hb ? __ldg(ep.bias + n + 1) : 0.0f, hb);
    if (ep.gelu) {
        y0 = gelu_pinned(y0);
        y1 = gelu_pinned(y1);
    }
    switch (ep.mode) {
    case OUT_F32: *reinterpret_cast<float2*>(orow + (int64_t)n * 4) = make_float2(y0, y1); break;
    case OUT_BF16: *reinterpret_cast<uint32_t*>(orow + (int64_t)n * 2) = pack_bf16x2(y0, y1); break;
    case OUT_F16: *reinterpret_cast<uint32_t*>(orow + (int64_t)n * 2) = pack_f16x2(y0, y1); break;
    case OUT_I4:
        orow[n >> 1] = (uint8_t)((quant_code(y0, ep.s_out, ep.qmin, ep.qmax) & 0xF) |
                                 ((quant_code(y1, ep.s_out, ep.qmin, ep.qmax) & 0xF) << 4));
        break;
    case OUT_I8:
        *reinterpret_cast<uint16_t*>(orow + n) =
            (uint16_t)((quant_code(y0, ep.s_out, ep.qmin, ep.qmax) & 0xFF) |
                       ((quant_code(y1, ep.s_out, ep.qmin, ep.qmax) & 0xFF) << 8));
        break;
    default: break;
    }
}

// grid: (n_tiles, m_tiles); a [M, K*bits/8] bytes row stride lda, w [N, ...].
template <bool kInt4>
__global__ void __launch_bounds__(kThreads) gemm_mma_small_kernel(const uint8_t* __restrict__ a, int64_t lda,
                                                                  const uint8_t* __restrict__ w, int64_t ldw,
                                                                  const EpiParams ep, int M, int N, int K) {
    asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory");   // PDL (ptx.cuh)
    using C = Cfg<kInt4>;
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;   // warp sub-tile
    const int64_t kbytes = kInt4 ? K / 2 : K;
    const int nkb = (K + BK - 1) / BK;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
    constexpr int kCpr = C::kRowBytes / 16;           // 16-byte chunks per tile row per stage
    constexpr int kChunks = (BM + BN) * kCpr;
    static_assert(kChunks % kThreads == 0, "chunk split");

    auto load_stage = [&](int kb, int slot) {
        const uint32_t base = s0 + slot * C::kStage;
#pragma unroll
        for (int i = 0; i < kChunks / kThreads; ++i) {
            const int id = tid + kThreads * i;
            const int r = id / kCpr, c = id % kCpr;
            const int64_t kofs = (int64_t)kb * C::kRowBytes + c * 16;
            const bool kin = kofs < kbytes;   // K % 32 == 0: chunks never straddle the end
            if (r < BM) {
                const int row = m0 + r;
                const bool v = kin && row < M;
                cp16(base + r * C::kPitch + c * 16, a + (int64_t)(v ? row : 0) * lda + (v ? kofs : 0), v);
            } else {
                const int row = n0 + (r - BM);
                const bool v = kin && row < N;
                cp16(base + r * C::kPitch + c * 16, w + (int64_t)(v ? row : 0) * ldw + (v ? kofs : 0), v);
            }
        }
    };

    int acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nkb) load_stage(s, s);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int kb = 0; kb < nkb; ++kb) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
        __syncthreads();
        {   // prefetch stage kb + kStages - 1 into the slot freed at kb - 1
            const int nk = kb + kStages - 1;
            if (nk < nkb) load_stage(nk, nk % kStages);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        const uint8_t* st = smem + (kb % kStages) * C::kStage;
        const uint8_t* As = st;
        const uint8_t* Ws = st + BM * C::kPitch;
#pragma unroll
        for (int ks = 0; ks < BK / 32; ++ks) {   // MMA K steps of 32 codes
            uint32_t af[2][4], bf[4][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int r = wm + 16 * i + g;
                if constexpr (kInt4) {   // word of codes [32ks + 8t, +8) of rows r, r+8
                    const uint32_t p0 = *reinterpret_cast<const uint32_t*>(As + r * C::kPitch + 16 * ks + 4 * t);
                    const uint32_t p1 = *reinterpret_cast<const uint32_t*>(As + (r + 8) * C::kPitch + 16 * ks + 4 * t);
                    af[i][0] = (p0 << 4) & 0xF0F0F0F0u; af[i][2] = p0 & 0xF0F0F0F0u;
                    af[i][1] = (p1 << 4) & 0xF0F0F0F0u; af[i][3] = p1 & 0xF0F0F0F0u;
                } else {
                    const uint8_t* q = As + r * C::kPitch + 32 * ks + 4 * t;
                    af[i][0] = *reinterpret_cast<const uint32_t*>(q);
                    af[i][1] = *reinterpret_cast<const uint32_t*>(q + 8 * C::kPitch);
                    af[i][2] = *reinterpret_cast<const uint32_t*>(q + 16);
                    af[i][3] = *reinterpret_cast<const uint32_t*>(q + 8 * C::kPitch + 16);
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = wn + 8 * j + g;
                if constexpr (kInt4) {
                    const uint32_t p = *reinterpret_cast<const uint32_t*>(Ws + r * C::kPitch + 16 * ks + 4 * t);
                    bf[j][0] = (p << 4) & 0xF0F0F0F0u;
                    bf[j][1] = p & 0xF0F0F0F0u;
                } else {
                    const uint8_t* q = Ws + r * C::kPitch + 32 * ks + 4 * t;
                    bf[j][0] = *reinterpret_cast<const uint32_t*>(q);
                    bf[j][1] = *reinterpret_cast<const uint32_t*>(q + 16);
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) imma(acc[i][j], af[i][0], af[i][1], af[i][2], af[i][3], bf[j][0], bf[j][1]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // ---- epilogue on the fragments: rows g / g+8, columns 2t, 2t+1 of each n8 tile
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int row = m0 + wm + 16 * i + g + 8 * h, n = n0 + wn + 8 * j + 2 * t;
                if (row < M && n < N) {
                    int32_t v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
                    if (kInt4) { v0 >>= 8; v1 >>= 8; }
                    emit2(ep, row, n, v0, v1);
                }
            }
}

}  // namespace gsm
}  // namespace mkq
