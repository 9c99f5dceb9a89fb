// quantize.cuh -- §8(a) rows a0 (weight calibration) and a1 (activation
// quantize + pack): HBM-bound elementwise kernels.
//
//   q = clamp(rint_even(x / s), qmin, qmax)        Eq.1, R1-R3
//   int4: byte k/2 of a row = (q[k] & 0xF) | (q[k+1] << 4)   (D2, R12)
//   s_w[n] = max(max_k |w[n,k]| / l_max, 1e-8)    P:72, R5/R6
#pragma once
#include <cstdint>
#include "epilogue.cuh"

namespace mkq {

// Fast path: every thread converts 8 consecutive elements of one row
// (2 x 128-bit loads -> one 32-bit store of 8 nibbles, or 64-bit of 8 bytes).
// Requires cols % 8 == 0, 16-byte aligned rows (ldx % 4 == 0) and aligned q.
template <int kBits, bool kPerRow>
__global__ void __launch_bounds__(256) quantize_pack_vec_kernel(
    const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
    const float* __restrict__ scale, float s_val, int qmin, int qmax, uint8_t* __restrict__ q, int64_t ldq) {
    asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory");   // PDL (ptx.cuh)
    const int64_t per_row = cols >> 3;
    const int64_t total = rows * per_row;
    const float s_t = (kPerRow || !scale) ? s_val : __ldg(scale);
    const QuantRcp Q_t = quant_rcp(s_t, qmin, qmax);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (!kPerRow) {
        // two groups per iteration: 4 x 16-byte loads in flight per thread
        for (; g + stride < total; g += 2 * stride) {
            const int64_t r0 = g / per_row, r1 = (g + stride) / per_row;
            const int64_t c0 = (g - r0 * per_row) << 3, c1 = (g + stride - r1 * per_row) << 3;
            const float4* s0p = reinterpret_cast<const float4*>(x + r0 * ldx + c0);
            const float4* s1p = reinterpret_cast<const float4*>(x + r1 * ldx + c1);
            const float4 a0 = __ldcs(s0p), b0 = __ldcs(s0p + 1), a1 = __ldcs(s1p), b1 = __ldcs(s1p + 1);
            const float v0[8] = {a0.x, a0.y, a0.z, a0.w, b0.x, b0.y, b0.z, b0.w};
            const float v1[8] = {a1.x, a1.y, a1.z, a1.w, b1.x, b1.y, b1.z, b1.w};
            if constexpr (kBits == 4) {
                // f32x2 reciprocal path; groups within 2^-18 of a rounding
                // boundary take the out-of-line exact Eq.1 (issue-bound
                // before: ncu issue 77%, profiles/r02_layer_kernels.md)
                bool n0 = false, n1 = false;
                uint32_t w0 = quant_nib8_fast(v0, Q_t, n0), w1 = quant_nib8_fast(v1, Q_t, n1);
                if (__builtin_expect(n0, 0)) w0 = quant_nib8_exact(v0[0], v0[1], v0[2], v0[3], v0[4], v0[5], v0[6], v0[7], s_t, qmin, qmax);
                if (__builtin_expect(n1, 0)) w1 = quant_nib8_exact(v1[0], v1[1], v1[2], v1[3], v1[4], v1[5], v1[6], v1[7], s_t, qmin, qmax);
                *reinterpret_cast<uint32_t*>(q + r0 * ldq + (c0 >> 1)) = w0;
                *reinterpret_cast<uint32_t*>(q + r1 * ldq + (c1 >> 1)) = w1;
            } else {
                int q0[8], q1[8];
                quant_group_rcp(v0, Q_t, q0);
                quant_group_rcp(v1, Q_t, q1);
                *reinterpret_cast<uint2*>(q + r0 * ldq + c0) =
                    make_uint2(pack_byte4(q0[0], q0[1], q0[2], q0[3]), pack_byte4(q0[4], q0[5], q0[6], q0[7]));
                *reinterpret_cast<uint2*>(q + r1 * ldq + c1) =
                    make_uint2(pack_byte4(q1[0], q1[1], q1[2], q1[3]), pack_byte4(q1[4], q1[5], q1[6], q1[7]));
            }
        }
    }
    for (; g < total; g += stride) {
        const int64_t r = g / per_row;
        const int64_t c8 = (g - r * per_row) << 3;
        const QuantRcp Q = kPerRow ? quant_rcp(__ldg(scale + r), qmin, qmax) : Q_t;
        const float4* src = reinterpret_cast<const float4*>(x + r * ldx + c8);
        const float4 a = __ldcs(src), b = __ldcs(src + 1);
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        int c[8];
        quant_group_rcp(v, Q, c);
        if constexpr (kBits == 4) {
            *reinterpret_cast<uint32_t*>(q + r * ldq + (c8 >> 1)) = pack_nib8(c);
        } else {
            uint2 w = make_uint2(pack_byte4(c[0], c[1], c[2], c[3]), pack_byte4(c[4], c[5], c[6], c[7]));
            *reinterpret_cast<uint2*>(q + r * ldq + c8) = w;
        }
    }
}

// General path: one thread per output byte (int4: 2 elements; int8: 1).
template <int kBits>
__global__ void __launch_bounds__(256) quantize_pack_any_kernel(
    const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
    const float* __restrict__ scale, float s_val, int per_row, int qmin, int qmax, uint8_t* __restrict__ q,
    int64_t ldq) {
    asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory");   // PDL (ptx.cuh)
    const int64_t per = kBits == 4 ? cols / 2 : cols;
    const int64_t total = rows * per;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / per, b = g - r * per;
        const float s = scale ? __ldg(scale + (per_row ? r : 0)) : s_val;
        if constexpr (kBits == 4) {
            const int lo = quant_code(x[r * ldx + 2 * b], s, qmin, qmax);
            const int hi = quant_code(x[r * ldx + 2 * b + 1], s, qmin, qmax);
            q[r * ldq + b] = (uint8_t)((lo & 0xF) | ((hi & 0xF) << 4));
        } else {
            q[r * ldq + b] = (uint8_t)(quant_code(x[r * ldx + b], s, qmin, qmax) & 0xFF);
        }
    }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Per-row max-abs (one warp per row, 128-bit loads when aligned, warp-shuffle
// reduction); writes s = max(absmax / l_max, 1e-8) (per_row) or folds the row
// maxima into *gmax_bits with an integer atomicMax on the (non-negative)
// float bit pattern (per-tensor).
__global__ void __launch_bounds__(256) absmax_rows_kernel(const float* __restrict__ x, int64_t rows,
                                                          int64_t cols, int64_t ldx, int vec,
                                                          float l_max, float* __restrict__ s_out,
                                                          unsigned int* gmax_bits) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const float* row = x + r * ldx;
        float m = 0.0f;
        if (vec) {
            for (int64_t c = lane * 4; c < cols; c += 128) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(row + c));
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
            }
        } else {
            for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, fabsf(row[c]));
        }
        m = warp_max(m);
        if (lane == 0) {
            if (s_out) {
                const float v = __fdiv_rn(m, l_max);
                s_out[r] = v < 1e-8f ? 1e-8f : v;
            } else {
                atomicMax(gmax_bits, __float_as_uint(m));
            }
        }
    }
}

__global__ void absmax_finalize_kernel(const unsigned int* gmax_bits, float l_max, float* s_out) {
    const float v = __fdiv_rn(__uint_as_float(*gmax_bits), l_max);
    s_out[0] = v < 1e-8f ? 1e-8f : v;
}

}  // namespace mkq

namespace mkq {
// Rank-major all-gather result [g][rows][cb] -> row-major [rows][g*cb]
// (column-parallel FFN: the FFN2 input codes / the FFN2 output columns).
// One thread per 16-byte chunk; cb % 16 == 0.
__global__ void __launch_bounds__(256) interleave_blocks_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                                int64_t g, int64_t rows, int64_t cb, int64_t ldd) {
    const int64_t cpr = cb / 16;                  // chunks per (rank, row)
    const int64_t total = g * rows * cpr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % cpr, rr = (i / cpr) % rows, r = i / (cpr * rows);
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src + (r * rows + rr) * cb) + c);
        *(reinterpret_cast<uint4*>(dst + rr * ldd + r * cb) + c) = v;
    }
}
}  // namespace mkq
