// attention.cuh -- §8(a) row a8 glue (★s): the multi-head self-attention
// core of Eq.3-5 (q.k^T per reading R8), softmax in fp32,
// fp16 operands (R10), fused with the Eq.1 quantize of OA for the W^A GEMM.
//
// One CTA = 64 query rows of one (sequence, head); 4 warps x 16 rows.
// K/V blocks of 64 keys stream through a double-buffered, XOR-swizzled
// shared-memory ring (cp.async); S = Q K^T and O += P V run on the tensor
// cores via mma.sync m16n8k16 (f16 x f16 -> f32) with an online (flash)
// softmax in fp32.  Sequences are packed back to back ("valid tokens",
// P:256, R13) and described by cu_seqlens.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "epilogue.cuh"

namespace mkq {
namespace attn {

constexpr int kD = 64;        // head_dim
constexpr int kBQ = 64;       // query rows per CTA
constexpr int kBK = 64;       // keys per block
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t swz(int row, int chunk) {   // byte offset in a 64x64 f16 tile
    return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* g, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem), "l"(g),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// Load a 64-row x 64-dim f16 tile (rows [r0, r0+64) of the sequence) into a
// swizzled smem tile; rows >= len are zero-filled.
__device__ __forceinline__ void load_tile(uint32_t sbase, const __half* g, int64_t ld, int r0, int len, int tid) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int id = tid + kThreads * i;   // 512 chunks of 16 B
        const int r = id >> 3, c = id & 7;
        const bool valid = (r0 + r) < len;
        const __half* src = g + (int64_t)(valid ? (r0 + r) : 0) * ld + c * 8;
        cp_async16(sbase + swz(r, c), src, valid);
    }
}

struct Params {
    const __half* qkv;
    int64_t ld;          // elements
    const int32_t* cu;   // [batch+1] or null
    int seq;             // fixed length when cu == null
    int hidden;          // heads * 64
    int out_mode;        // 0 f32, 3 int4, 4 int8
    float s_out;
    int qmin, qmax;
    void* out;
    int64_t ldo;         // bytes
};

__global__ void __launch_bounds__(kThreads) flash_attn_kernel(const Params p) {
    asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory");   // PDL (ptx.cuh)
    __shared__ __align__(128) uint8_t smem[kBQ * 128 + 4 * kBK * 128];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int head = blockIdx.y, b = blockIdx.z;
    const int start = p.cu ? p.cu[b] : b * p.seq;
    const int len = p.cu ? (p.cu[b + 1] - start) : p.seq;
    const int q0 = blockIdx.x * kBQ;
    if (q0 >= len) return;

    const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sK[2] = {sQ + kBQ * 128, sQ + kBQ * 128 + kBK * 128};
    const uint32_t sV[2] = {sQ + kBQ * 128 + 2 * kBK * 128, sQ + kBQ * 128 + 3 * kBK * 128};

    const __half* base = p.qkv + (int64_t)start * p.ld + head * kD;
    const __half* gQ = base;
    const __half* gK = base + p.hidden;
    const __half* gV = base + 2 * p.hidden;

    load_tile(sQ, gQ, p.ld, q0, len, tid);
    load_tile(sK[0], gK, p.ld, 0, len, tid);
    load_tile(sV[0], gV, p.ld, 0, len, tid);
    cp_async_commit();

    const int nblk = (len + kBK - 1) / kBK;
    const float scale_log2 = 0.125f * 1.4426950408889634f;   // 1/sqrt(64) * log2(e)
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
    float o[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    uint32_t qa[4][4];   // Q fragments for the 4 k16 steps over head_dim

    for (int kb = 0; kb < nblk; ++kb) {
        const int cur = kb & 1;
        if (kb + 1 < nblk) {
            load_tile(sK[cur ^ 1], gK, p.ld, (kb + 1) * kBK, len, tid);
            load_tile(sV[cur ^ 1], gV, p.ld, (kb + 1) * kBK, len, tid);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int r = warp * 16 + (lane & 15);
                const int c = kk * 2 + (lane >> 4);
                ldsm_x4(sQ + swz(r, c), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
            }
        }
        // ---- S = Q K^T  (16 rows x 64 keys per warp)
        float s[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int np = 0; np < 4; ++np) {   // pairs of n8 tiles (16 keys)
                const int key = np * 16 + (lane & 7) + 8 * (lane >> 4);
                const int c = kk * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sK[cur] + swz(key, c), b0, b1, b2, b3);
                mma16816(s[2 * np], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                mma16816(s[2 * np + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
            }
        }
        // ---- mask keys beyond the sequence, online softmax (fp32)
        const int kbase = kb * kBK;
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = kbase + i * 8 + 2 * (lane & 3) + (j & 1);
                float v = s[i][j] * scale_log2;
                if (key >= len) v = -INFINITY;
                s[i][j] = v;
                mx[j >> 1] = fmaxf(mx[j >> 1], v);
            }
        }
        float corr[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
            const float mnew = fmaxf(m_r[h], mx[h]);
            corr[h] = ex2(m_r[h] - mnew);
            m_r[h] = mnew;
            l_r[h] *= corr[h];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            o[i][0] *= corr[0]; o[i][1] *= corr[0];
            o[i][2] *= corr[1]; o[i][3] *= corr[1];
        }
        float rs[2] = {0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float e = ex2(s[i][j] - m_r[j >> 1]);
                s[i][j] = e;
                rs[j >> 1] += e;
            }
        }
        l_r[0] += rs[0];
        l_r[1] += rs[1];
        // ---- O += P V
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {   // 16 keys per step
            const uint32_t a0 = pack_h2(s[2 * kk][0], s[2 * kk][1]);
            const uint32_t a1 = pack_h2(s[2 * kk][2], s[2 * kk][3]);
            const uint32_t a2 = pack_h2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
            const uint32_t a3 = pack_h2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
            for (int np = 0; np < 4; ++np) {   // pairs of 8-dim output tiles
                const int key = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
                const int c = np * 2 + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(sV[cur] + swz(key, c), b0, b1, b2, b3);
                mma16816(o[2 * np], a0, a1, a2, a3, b0, b1);
                mma16816(o[2 * np + 1], a0, a1, a2, a3, b2, b3);
            }
        }
        __syncthreads();
    }
    // ---- finalize: O / l, store fp32 or quantized codes
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
        l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
    }
    const float inv[2] = {1.0f / l_r[0], 1.0f / l_r[1]};
    const QuantRcp Qo = quant_rcp(p.out_mode ? p.s_out : 1.0f, p.qmin, p.qmax);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = q0 + warp * 16 + (lane >> 2) + 8 * h;
        if (r >= len) continue;
        uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)(start + r) * p.ldo;
        float v[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            v[2 * i] = o[i][2 * h] * inv[h];
            v[2 * i + 1] = o[i][2 * h + 1] * inv[h];
        }
        if (p.out_mode == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                *reinterpret_cast<float2*>(orow + (int64_t)(head * kD + i * 8 + 2 * (lane & 3)) * 4) =
                    make_float2(v[2 * i], v[2 * i + 1]);
        } else {
            // Eq.1 via the reciprocal, the exact division only for a group with a
            // value near a rounding boundary (epilogue.cuh; was 16 IEEE divisions)
            int cq[16];
            quant_group_rcp(v, Qo, cq);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int col = head * kD + i * 8 + 2 * (lane & 3);
                const int c0 = cq[2 * i], c1 = cq[2 * i + 1];
                if (p.out_mode == 3) {
                    orow[col >> 1] = (uint8_t)((c0 & 0xF) | ((c1 & 0xF) << 4));
                } else {
                    *reinterpret_cast<uint16_t*>(orow + col) = (uint16_t)((c0 & 0xFF) | ((c1 & 0xFF) << 8));
                }
            }
        }
    }
}

}  // namespace attn
}  // namespace mkq
