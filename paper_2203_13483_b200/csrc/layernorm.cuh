// layernorm.cuh -- §8(a) row a8 glue (★s): residual + post-LayerNorm in fp32
// ("layernorm ... computed using float32"; R9 post-LN, eps 1e-12),
// optionally fused with the Eq.1 quantize of the normalised row (a1), so the
// LN output is never re-read from HBM just to be quantized.
//
// One warp per row; 128-bit loads; the row stays in registers between the
// mean pass, the centred-variance pass and the output pass; warp-shuffle
// reductions.
#pragma once
#include <cstdint>
#include "epilogue.cuh"

namespace mkq {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// VPL: float4 vectors per lane (cols <= 128*VPL).  kPre: gamma/beta issued
// together with the row loads (one memory round trip instead of two): used
// for small row counts (latency-bound); at large row counts the extra
// registers cost occupancy and bandwidth (measured 304 -> 439 us).
template <int VPL, bool kPre = false>
__global__ void __launch_bounds__(256) residual_ln_kernel(
    const float* __restrict__ x, const float* __restrict__ res, int64_t rows, int cols, int64_t ld,
    const float* __restrict__ g, const float* __restrict__ b, float eps, float* __restrict__ y,
    int bits, float s_q, int qmin, int qmax, uint8_t* __restrict__ q, int64_t ldq) {
    asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory");   // PDL (ptx.cuh)
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int nv = cols >> 2;
    const QuantRcp Qr = quant_rcp(s_q, qmin, qmax);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const float4* xr = reinterpret_cast<const float4*>(x + r * ld);
        const float4* rr = res ? reinterpret_cast<const float4*>(res + r * ld) : nullptr;
        float4 v[VPL], gg[kPre ? VPL : 1], bb[kPre ? VPL : 1];
        float s = 0.f;
        if constexpr (kPre) {
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                const int c = lane + 32 * i;
                if (c < nv) {
                    gg[i] = __ldg(reinterpret_cast<const float4*>(g) + c);
                    bb[i] = __ldg(reinterpret_cast<const float4*>(b) + c);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            const int c = lane + 32 * i;
            if (c < nv) {
                float4 a = __ldcs(xr + c);
                if (rr) {
                    const float4 t = __ldcs(rr + c);
                    a.x += t.x; a.y += t.y; a.z += t.z; a.w += t.w;
                }
                v[i] = a;
                s += (a.x + a.y) + (a.z + a.w);
            } else {
                v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const float mean = warp_sum(s) / (float)cols;
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            const int c = lane + 32 * i;
            if (c < nv) {
                const float dx = v[i].x - mean, dy = v[i].y - mean, dz = v[i].z - mean, dw = v[i].w - mean;
                ss += (dx * dx + dy * dy) + (dz * dz + dw * dw);
            }
        }
        const float rstd = rsqrtf(warp_sum(ss) / (float)cols + eps);
        float4* yr = reinterpret_cast<float4*>(y + r * ld);
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            const int c = lane + 32 * i;
            if (c < nv) {
                const float4 g4 = kPre ? gg[kPre ? i : 0] : __ldg(reinterpret_cast<const float4*>(g) + c);
                const float4 b4 = kPre ? bb[kPre ? i : 0] : __ldg(reinterpret_cast<const float4*>(b) + c);
                float4 o;
                o.x = (v[i].x - mean) * rstd * g4.x + b4.x;
                o.y = (v[i].y - mean) * rstd * g4.y + b4.y;
                o.z = (v[i].z - mean) * rstd * g4.z + b4.z;
                o.w = (v[i].w - mean) * rstd * g4.w + b4.w;
                yr[c] = o;
                if (bits) {
                    const float ov[4] = {o.x, o.y, o.z, o.w};
                    int cq[4];
                    quant_group_rcp(ov, Qr, cq);
                    if (bits == 4) {
                        const uint16_t w = (uint16_t)((cq[0] & 0xF) | ((cq[1] & 0xF) << 4) | ((cq[2] & 0xF) << 8) |
                                                      ((cq[3] & 0xF) << 12));
                        *reinterpret_cast<uint16_t*>(q + r * ldq + 2 * c) = w;
                    } else {
                        *reinterpret_cast<uint32_t*>(q + r * ldq + 4 * c) = pack_byte4(cq[0], cq[1], cq[2], cq[3]);
                    }
                }
            }
        }
    }
}

}  // namespace mkq
