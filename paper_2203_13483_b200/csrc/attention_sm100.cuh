// attention_sm100.cuh -- shared pieces of the §8(a) row a8 tcgen05 attention
// (Eq.3-5, q k^T per R8; fp16 operands, fp32 softmax per P:234):
// the work-item parameters, the kind::f16 MMA / instruction descriptors for
// Q K^T (SS) and P V (P from TMEM, TS), TMEM stores, and the FMA-pipe exp2
// polynomial.  The kernel using them is attn_pp_kernel
// (attention_pp_sm100.cuh); the earlier one-tile-per-CTA kernel built on them
// was superseded by it and removed.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include "epilogue.cuh"
#include "ptx.cuh"

namespace mkq {
namespace attn2 {

constexpr int kBQ = 128, kBK = 64, kD = 64;
constexpr int kStages = 3;
constexpr int kQBytes = kBQ * kD * 2;      // 16 KB
constexpr int kKVBytes = kBK * kD * 2;     // 8 KB (one K or V block)
constexpr int kSoftWarps = 8;              // 2 per TMEM lane quadrant, each half of the keys / O dims
constexpr int kThreads = 32 * (2 + kSoftWarps);   // warp 0 TMA + TMEM alloc, warp 1 MMA, warps 2-9 softmax
constexpr int kTmemCols = 256;             // S[0], S[1] (kBK each) + O (64): 2 CTAs per SM
constexpr float kRescale = 8.0f;           // lazy rescale threshold (log2): P <= 2^8 in fp16
constexpr int kXchg = 2 * 2 * kBQ * 4;     // partial row maxima [block parity][half][row]
constexpr int kSmem = 1024 + 2 * kQBytes + 2 * kStages * kKVBytes + kXchg + 256;

struct Params {
    const int32_t* cu;   // [batch+1] or null
    int seq;             // fixed length when cu == null
    int hidden;          // heads * 64
    int out_mode;        // 0 f32, 3 int4, 4 int8
    float s_out;
    int qmin, qmax;
    void* out;
    int64_t ldo;         // bytes
};

// kind::f16 instruction descriptor: D f32, A/B f16, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N, uint32_t b_mn_major) {
    return (1u << 4) | (b_mn_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// MN-major SW128 smem descriptor: 8 x 16-byte chunks along N per 128-byte
// row, rows along K; SBO = 1024 B between 8-row groups along K.
__device__ __forceinline__ uint64_t desc_sw128_mnmajor(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
    d |= (uint64_t)(1024 >> 4) << 16;    // LBO (stride between 64-element N atoms; one atom here)
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO: 8 K-rows x 128 B
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

// Warp-collective MMA issue (all lanes converged, elect.sync picks the issuer).
__device__ __forceinline__ void mma_f16_ss_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_f16_ts_warp(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// exp2 on the FMA/ALU pipes (offloads the MUFU/XU pipe, which bounds the
// softmax): 2^x = 2^n * p(f), n = rint(x) via the 1.5*2^23 magic add,
// f = x - n in [-0.5, 0.5], p a degree-3 minimax polynomial (max rel. error
// 1.0e-4 < the fp16 rounding of P), 2^n applied by adding n to the exponent
// field.  x is clamped at -125 so the exponent stays normal.
__device__ __forceinline__ float ex2_fma(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;
    const float n = t - 12582912.0f;
    const float f = x - n;
    float p = 0x1.ca1d02p-5f;
    p = fmaf(p, f, 0x1.f0ed48p-3f);
    p = fmaf(p, f, 0x1.62e0c2p-1f);
    p = fmaf(p, f, 0x1.fff61ap-1f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// packed fp32 pairs (sm_100 f32x2: one instruction, two IEEE RN results)
__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<const uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<const float2*>(&a); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
// ex2_fma on a pair, in f32x2 arithmetic (6 pair-ops + 2 clamps + 2 IMAD)
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
    x.x = fmaxf(x.x, -125.0f);
    x.y = fmaxf(x.y, -125.0f);
    const float2 t = fadd2(x, make_float2(12582912.0f, 12582912.0f));
    const float2 n = fadd2(t, make_float2(-12582912.0f, -12582912.0f));
    const float2 f = ffma2(n, make_float2(-1.0f, -1.0f), x);
    float2 p = ffma2(make_float2(0x1.ca1d02p-5f, 0x1.ca1d02p-5f), f, make_float2(0x1.f0ed48p-3f, 0x1.f0ed48p-3f));
    p = ffma2(p, f, make_float2(0x1.62e0c2p-1f, 0x1.62e0c2p-1f));
    p = ffma2(p, f, make_float2(0x1.fff61ap-1f, 0x1.fff61ap-1f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ uint32_t h2(float a, float b) {
    __half2 v = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace attn2
}  // namespace mkq
