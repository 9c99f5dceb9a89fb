// qat.cuh -- SURVEY §8(f) NEXT(3): the QAT-side kernels of §4.1.
//
// One HBM-bound pass over a tensor x with a learned per-tensor scale s:
//   q_i   = clamp(rint_even(x_i / s), qmin, qmax)          Eq.1, R1-R3
//   y_i   = fl32(s * q_i)                                   fake-quant Q[x]
//   clip_i= rint(x_i/s) outside [qmin, qmax]                R18
//   gx_i  = clip_i ? 0 : gy_i                               STE input gradient (R18)
//   STE   = sum_i (clip_i ? q_i : q_i - x_i/s)              P:138-142 + LSQ rule, R17
//   MSE   = 2 sum_i (s q_i - x_i) q_i
// The two reductions are carried as four sums that need no division per
// element:  Sq = sum q_i (exact int64), Sqq = sum q_i^2 (exact int64),
// Sxin = sum_{not clipped} x_i (fp64), Sxq = sum x_i q_i (fp64; each product
// is exact in fp64), then STE = Sq - Sxin/s and MSE = 2 (s Sqq - Sxq).
// Per-block partials go to a workspace and one block folds them in a fixed
// order, so the result is deterministic run to run.  The fp64 sums differ
// from the oracle's term-by-term sum only by rounding order.
#pragma once
#include <cstdint>
#include "epilogue.cuh"

namespace mkq {
namespace qat {

constexpr int kThreads = 256;

struct Partial {
    double sxin, sxq;
    long long sq, sqq;
};

// Unclamped code of x (clamped to [qmin-1, qmax+1], which keeps the magic-add
// rounding exact and preserves "outside [qmin, qmax]") via the reciprocal
// with one remainder correction; near a half-integer the exact IEEE
// division decides (same scheme as quant_code_rcp, epilogue.cuh).
__device__ __forceinline__ int code_unclamped(float x, const QuantRcp& Q) {
    float q = __fmul_rn(x, Q.r);
    const float rem = __fmaf_rn(-q, Q.s, x);
    q = __fmaf_rn(rem, Q.r, q);
    q = fminf(fmaxf(q, Q.lo - 1.0f), Q.hi + 1.0f);
    const float t = __fadd_rn(q, 12582912.0f);
    const float d = __fsub_rn(q, __fsub_rn(t, 12582912.0f));
    if (fabsf(__fsub_rn(fabsf(d), 0.5f)) <= __fmul_rn(fabsf(q), 0x1p-20f) + 0x1p-20f) {
        float v = __fdiv_rn(x, Q.s);
        v = fminf(fmaxf(v, Q.lo - 1.0f), Q.hi + 1.0f);
        return __float2int_rn(v);
    }
    return __float_as_int(t) - 0x4B400000;
}

struct Acc {
    double sxin = 0.0, sxq = 0.0;
    int sq = 0, sqq = 0;   // per-thread: |q| <= 128, <= 2^14 per element; flushed to 64-bit per chunk
};

__device__ __forceinline__ float one(float x, float gy, const QuantRcp& Q, Acc& a, float& gx) {
    const int r = code_unclamped(x, Q);
    const bool clip = r < Q.qmin || r > Q.qmax;
    const int q = min(max(r, Q.qmin), Q.qmax);
    a.sq += q;
    a.sqq += q * q;
    a.sxq = fma((double)x, (double)q, a.sxq);
    if (!clip) a.sxin += (double)x;
    gx = clip ? 0.0f : gy;
    return __fmul_rn(Q.s, (float)q);
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    T t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : T(0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;   // valid in thread 0
}

// Grid-stride over 4-element chunks; `vec` = every pointer 16-byte aligned.
__global__ void __launch_bounds__(kThreads) fake_quant_grad_kernel(
    const float* __restrict__ x, int64_t n, const float* __restrict__ scale, int qmin, int qmax,
    float* __restrict__ y, const float* __restrict__ gy, float* __restrict__ gx, Partial* __restrict__ part,
    int vec) {
    const QuantRcp Q = quant_rcp(__ldg(scale), qmin, qmax);
    Acc a;
    long long sq = 0, sqq = 0;
    const int64_t chunks = (n + 3) >> 2;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = c << 2;
        if (vec && i0 + 4 <= n) {
            const float4 xv = __ldcs(reinterpret_cast<const float4*>(x + i0));
            float4 gv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gy) gv = __ldcs(reinterpret_cast<const float4*>(gy + i0));
            float4 yv, gxv;
            yv.x = one(xv.x, gv.x, Q, a, gxv.x);
            yv.y = one(xv.y, gv.y, Q, a, gxv.y);
            yv.z = one(xv.z, gv.z, Q, a, gxv.z);
            yv.w = one(xv.w, gv.w, Q, a, gxv.w);
            if (y) __stcs(reinterpret_cast<float4*>(y + i0), yv);
            if (gx) __stcs(reinterpret_cast<float4*>(gx + i0), gxv);
        } else {
            for (int64_t i = i0; i < n && i < i0 + 4; ++i) {
                float g;
                const float v = one(x[i], gy ? gy[i] : 0.0f, Q, a, g);
                if (y) y[i] = v;
                if (gx) gx[i] = g;
            }
        }
        sq += a.sq;
        sqq += a.sqq;
        a.sq = a.sqq = 0;
    }
    __shared__ double shd[kThreads / 32];
    __shared__ long long shl[kThreads / 32];
    Partial p;
    p.sxin = block_sum(a.sxin, shd);
    p.sxq = block_sum(a.sxq, shd);
    p.sq = block_sum(sq, shl);
    p.sqq = block_sum(sqq, shl);
    if (threadIdx.x == 0) part[blockIdx.x] = p;
}

// One block folds the per-block partials in index order (deterministic) and
// writes grad_s = {STE, MSE}.
__global__ void __launch_bounds__(kThreads) fake_quant_finalize_kernel(const Partial* __restrict__ part, int nparts,
                                                                       const float* __restrict__ scale,
                                                                       double* __restrict__ grad_s) {
    double sxin = 0.0, sxq = 0.0;
    long long sq = 0, sqq = 0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
        sxin += part[i].sxin;
        sxq += part[i].sxq;
        sq += part[i].sq;
        sqq += part[i].sqq;
    }
    __shared__ double shd[kThreads / 32];
    __shared__ long long shl[kThreads / 32];
    sxin = block_sum(sxin, shd);
    sxq = block_sum(sxq, shd);
    sq = block_sum(sq, shl);
    sqq = block_sum(sqq, shl);
    if (threadIdx.x == 0) {
        const double s = (double)__ldg(scale);
        grad_s[0] = (double)sq - sxin / s;
        grad_s[1] = 2.0 * (s * (double)sqq - sxq);
    }
}

}  // namespace qat
}  // namespace mkq
