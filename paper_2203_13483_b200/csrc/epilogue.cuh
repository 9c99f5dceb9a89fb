// epilogue.cuh -- per-element arithmetic of the fused GEMM epilogue (§8a rows
// a4 dequant, a5 GELU, a6 requantize) and of the activation quantizer (a1).
//
// Every sequence below is pinned by a DESIGN.md reading so that the CUDA
// path and the CPU oracle compute the same binary32 values:
//   R2/R3  quantize : q = clamp(rint_even(x / s)), one IEEE division
//   R4     dequant  : sc = fl(s_a*s_w[n]); y = fma((float)acc, sc, b[n])
//   R7     gelu     : 0.5*y*(1+erf_pinned(|y|/sqrt2)) with the frozen erf
//                     polynomial (hex-exact binary32 constants, R7)
//   R11    bf16/f16 : round-to-nearest-even of the fp32 value
// Explicit __f*_rn intrinsics keep nvcc from contracting or reordering.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace mkq {

// Eq.1: clamp(round(x/s)), ties to even, fp32 division.
__device__ __forceinline__ int quant_code(float x, float s, int qmin, int qmax) {
    int q = __float2int_rn(__fdiv_rn(x, s));
    return min(max(q, qmin), qmax);
}

// Eq.1 without a division per element, for epilogues that quantize many
// values by one scale: q = x*r corrected once by the remainder
// (r = RN(1/s); rem = x - q*s is exact in the fma; q' = q + rem*r), clamped
// to [qmin, qmax] (clamp and rint commute for integer bounds) and rounded
// with the 1.5*2^23 magic add (exact for |q| <= 2^22).  q' is within an ulp
// or two of x/s, so its code can differ from quant_code's only when q' lies
// within a few ulps of a half-integer rounding boundary: `near` reports that
// case and the caller recomputes those values with quant_code (rare).
struct QuantRcp {
    float s, r, lo, hi;
    int qmin, qmax;
};
__device__ __forceinline__ QuantRcp quant_rcp(float s, int qmin, int qmax) {
    return QuantRcp{s, __frcp_rn(s), (float)qmin, (float)qmax, qmin, qmax};
}
__device__ __forceinline__ int quant_code_rcp(float x, const QuantRcp& Q, bool& near) {
    float q = __fmul_rn(x, Q.r);
    const float rem = __fmaf_rn(-q, Q.s, x);
    q = __fmaf_rn(rem, Q.r, q);
    q = fminf(fmaxf(q, Q.lo), Q.hi);   // NaN -> lo, like quant_code
    const float t = __fadd_rn(q, 12582912.0f);
    const float d = __fsub_rn(q, __fsub_rn(t, 12582912.0f));   // q - rint(q), in [-0.5, 0.5]
    near |= fabsf(__fsub_rn(fabsf(d), 0.5f)) <= __fmul_rn(fabsf(q), 0x1p-20f);
    return __float_as_int(t) - 0x4B400000;
}

// A group of codes with one near-boundary check (the exact fallback is taken
// for the whole group, keeping the common path branch-free).
template <int N>
__device__ __forceinline__ void quant_group_rcp(const float (&v)[N], const QuantRcp& Q, int (&c)[N]) {
    bool near = false;
#pragma unroll
    for (int i = 0; i < N; ++i) c[i] = quant_code_rcp(v[i], Q, near);
    if (near) {
#pragma unroll
        for (int i = 0; i < N; ++i) c[i] = quant_code(v[i], Q.s, Q.qmin, Q.qmax);
    }
}

// Out-of-line exact fallbacks for code-size-sensitive epilogues (the
// near-boundary case is rare; keeping the IEEE divisions out of line keeps
// the hot loop in the instruction cache).
__device__ __noinline__ uint32_t quant_nib8_exact(float v0, float v1, float v2, float v3, float v4, float v5, float v6,
                                                  float v7, float s, int qmin, int qmax) {
    const float v[8] = {v0, v1, v2, v3, v4, v5, v6, v7};
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint32_t)(quant_code(v[i], s, qmin, qmax) & 0xF) << (4 * i);
    return w;
}
__device__ __noinline__ uint32_t quant_byte4_exact(float v0, float v1, float v2, float v3, float s, int qmin, int qmax) {
    return (uint32_t)(quant_code(v0, s, qmin, qmax) & 0xFF) | ((uint32_t)(quant_code(v1, s, qmin, qmax) & 0xFF) << 8) |
           ((uint32_t)(quant_code(v2, s, qmin, qmax) & 0xFF) << 16) | ((uint32_t)(quant_code(v3, s, qmin, qmax) & 0xFF) << 24);
}
__device__ __forceinline__ uint32_t quant_nib8_rcp(const float (&v)[8], const QuantRcp& Q) {
    bool near = false;
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint32_t)(quant_code_rcp(v[i], Q, near) & 0xF) << (4 * i);
    if (near) w = quant_nib8_exact(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], Q.s, Q.qmin, Q.qmax);
    return w;
}
__device__ __forceinline__ uint32_t quant_byte4_rcp(float v0, float v1, float v2, float v3, const QuantRcp& Q) {
    bool near = false;
    const int c0 = quant_code_rcp(v0, Q, near), c1 = quant_code_rcp(v1, Q, near);
    const int c2 = quant_code_rcp(v2, Q, near), c3 = quant_code_rcp(v3, Q, near);
    if (near) return quant_byte4_exact(v0, v1, v2, v3, Q.s, Q.qmin, Q.qmax);
    return (uint32_t)(c0 & 0xFF) | ((uint32_t)(c1 & 0xFF) << 8) | ((uint32_t)(c2 & 0xFF) << 16) | ((uint32_t)(c3 & 0xFF) << 24);
}

// f32x2 arithmetic (sm_100: two IEEE RN fp32 operations per instruction)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {   // two IEEE RN fmas, one instruction
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)),
          "l"(*reinterpret_cast<const uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {   // two IEEE RN adds, one instruction
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {   // two IEEE RN multiplies, one instruction
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
    return *reinterpret_cast<float2*>(&r);
}

// Eq.1 codes of 8 values with one scale, int4 nibbles packed (value i in
// nibble i), for epilogues where |code| is small: q = fl(x * RN(1/s)) differs
// from fl(x / s) by at most 2 ulps of |q| <= 2^-19 inside the code range
// [qmin, qmax] (|q| <= 8 after the clamp), so rint(clamp(q)) equals Eq.1's
// rint(clamp(fl(x/s))) unless q lies within 2^-18 of a half-integer, which the
// caller's `near` reports (evaluate those groups with quant_code).  Clamping
// before rounding is rounding before clamping for integer bounds.
__device__ __forceinline__ uint32_t quant_nib8_fast(const float (&x)[8], const QuantRcp& Q, bool& near) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        float2 q = mul2(make_float2(x[i], x[i + 1]), make_float2(Q.r, Q.r));
        q.x = fminf(fmaxf(q.x, Q.lo), Q.hi);
        q.y = fminf(fmaxf(q.y, Q.lo), Q.hi);
        const float2 t = add2(q, make_float2(12582912.0f, 12582912.0f));
        const float2 d = fma2(add2(t, make_float2(-12582912.0f, -12582912.0f)), make_float2(-1.0f, -1.0f), q);
        near |= fabsf(fabsf(d.x) - 0.5f) <= 0x1p-18f;
        near |= fabsf(fabsf(d.y) - 0.5f) <= 0x1p-18f;
        w |= ((__float_as_uint(t.x) & 0xFu) << (4 * i)) | ((__float_as_uint(t.y) & 0xFu) << (4 * i + 4));
    }
    return w;
}

// Dequant (P:66 s*q, P:93/P:98 bias; reading R4).
__device__ __forceinline__ float dequant(int32_t acc, float sc, float b, bool has_bias) {
    float a = __int2float_rn(acc);
    return has_bias ? __fmaf_rn(a, sc, b) : __fmul_rn(a, sc);
}

// gelu_pinned (P:98 GELU, computed in float32 per P:234; reading R7).
// erf piece 1 (t < 1): t * P(t^2), P degree 6; piece 2 (1 <= t < 3.92):
// 1 - Q(t - 2.5), Q degree 12; t >= 3.92: 1.  Both pieces are evaluated
// and selected (branch-free across a warp).
__device__ __forceinline__ float gelu_pinned(float y) {
    const float t = __fmul_rn(fabsf(y), 0x1.6a09e6p-1f);
    const float u1 = __fmul_rn(t, t);
    float p = 0x1.4fd528p-14f;
    p = __fmaf_rn(p, u1, -0x1.a63f9ep-11f);
    p = __fmaf_rn(p, u1, 0x1.545360p-8f);
    p = __fmaf_rn(p, u1, -0x1.b80286p-6f);
    p = __fmaf_rn(p, u1, 0x1.ce2d7cp-4f);
    p = __fmaf_rn(p, u1, -0x1.812740p-2f);
    p = __fmaf_rn(p, u1, 0x1.20dd76p+0f);
    const float e1 = __fmul_rn(t, p);
    const float u2 = __fsub_rn(t, 2.5f);
    float q = 0x1.3db5fep-17f;
    q = __fmaf_rn(q, u2, -0x1.5d0ec2p-16f);
    q = __fmaf_rn(q, u2, -0x1.0bd2eep-14f);
    q = __fmaf_rn(q, u2, 0x1.23355ep-12f);
    q = __fmaf_rn(q, u2, -0x1.280846p-12f);
    q = __fmaf_rn(q, u2, -0x1.29eb5ap-11f);
    q = __fmaf_rn(q, u2, 0x1.70d992p-9f);
    q = __fmaf_rn(q, u2, -0x1.901754p-8f);
    q = __fmaf_rn(q, u2, 0x1.1a5d5cp-7f);
    q = __fmaf_rn(q, u2, -0x1.11b3b0p-7f);
    q = __fmaf_rn(q, u2, 0x1.64ef0ap-8f);
    q = __fmaf_rn(q, u2, -0x1.1d7db8p-9f);
    q = __fmaf_rn(q, u2, 0x1.aab4b4p-12f);
    const float e2 = __fsub_rn(1.0f, q);
    float e = (t < 1.0f) ? e1 : ((t < 3.92f) ? e2 : 1.0f);
    e = (y < 0.0f) ? -e : e;
    const float h = __fmul_rn(0.5f, y);
    return __fmaf_rn(h, e, h);
}

__device__ __forceinline__ uint32_t pack_nib8(const int (&q)[8]) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint32_t)(q[i] & 0xF) << (4 * i);
    return w;
}

__device__ __forceinline__ uint32_t pack_byte4(int a, int b, int c, int d) {
    return (uint32_t)(a & 0xFF) | ((uint32_t)(b & 0xFF) << 8) | ((uint32_t)(c & 0xFF) << 16) |
           ((uint32_t)(d & 0xFF) << 24);
}

// R11: round-to-nearest-even of each fp32 value, a in the low half: one
// cvt.rn.*x2.f32 (F2FP.PACK_AB) per pair instead of two scalar conversions
// through the MIO pipe (the QKV epilogue's top stall in the r02 profile)
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

}  // namespace mkq
