// attention_sm100.cuh -- §8(a) row a8 glue: multi-head self-attention core of
// Eq.3-5 (q k^T per R8) on the 5th-generation tensor cores, fp16
// operands (R10), fp32 softmax, fused Eq.1 quantize of OA (a1).
//
// One CTA = 128 query rows of one (sequence, head):
//   warp 0      TMA: Q tile once, then K_j / V_j (64 keys x 64 dims, fp16,
//               SWIZZLE_128B) through a 3-stage ring
//   warp 1      MMA issuer:  S_j = Q K_j^T  (tcgen05.mma kind::f16, M=128,
//               N=64, fp32 accumulate, TMEM, double-buffered)
//               O += P_j V_j (A = P_j read from TMEM, B = V_j MN-major smem)
//   warps 2-9   softmax / correction / epilogue: two warps per query row
//               group (each half of the keys and of the O dims);
//               tcgen05.ld S_j row -> online max/sum in fp32 -> P_j (fp16)
//               tcgen05.st back over S_j's columns -> rescale O in TMEM when
//               the running max moved -> after the last block O/l ->
//               quantize -> int4/int8 codes (or fp32) to global memory.
// TMEM: S[0] cols [0,64), S[1] [64,128), O [128,192) (alloc 256: two CTAs per
// SM, so one CTA's TMA/softmax latency overlaps the other's MMAs).  O
// accumulates in TMEM across key blocks; the exponentials use a reference max
// that is only raised (and O, l rescaled) when a block's max exceeds it by
// more than 2^8 (lazy rescaling: P <= 256 stays exact enough in fp16, and
// with BERT-like scores the reference rarely moves after the first block).
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

struct Item {
    int start, len, head, q0, nblk;
};

__device__ __forceinline__ bool get_item(const Params& p, int w, int heads, int qtiles, Item& it) {
    const int qt = w % qtiles;
    const int bh = w / qtiles;
    const int h = bh % heads, b = bh / heads;
    it.start = p.cu ? p.cu[b] : b * p.seq;
    it.len = p.cu ? (p.cu[b + 1] - it.start) : p.seq;
    it.head = h;
    it.q0 = qt * kBQ;
    it.nblk = (it.len + kBK - 1) / kBK;
    return it.q0 < it.len;
}

// Persistent: each CTA walks work items w = blockIdx.x + i*gridDim.x over
// (sequence, head, 128-query tile); the K/V ring, the S/O buffers and their
// barrier phases run on one block counter g across items, so the next item's
// Q/K/V loads and first S MMA overlap the current item's tail.
__global__ void __launch_bounds__(kThreads, 2)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const Params p, int heads, int qtiles, int nitems) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                             // 2 tiles
    uint8_t* sK = sQ + 2 * kQBytes;                 // kStages tiles
    uint8_t* sV = sK + kStages * kKVBytes;          // kStages tiles
    float* xchg = reinterpret_cast<float*>(sV + kStages * kKVBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xchg) + kXchg);
    uint64_t* q_full = bars;                        // [2]
    uint64_t* q_empty = q_full + 2;                 // [2]
    uint64_t* k_full = q_empty + 2;                 // [kStages]
    uint64_t* v_full = k_full + kStages;            // [kStages]
    uint64_t* kv_empty = v_full + kStages;          // [kStages]
    uint64_t* s_full = kv_empty + kStages;          // [2]
    uint64_t* p_ready = s_full + 2;                 // [2]
    uint64_t* pv_done = p_ready + 2;                // [2] (by block parity)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&q_full[i], 1);
            ptx::mbar_init(&q_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&p_ready[i], kSoftWarps);
            ptx::mbar_init(&pv_done[i], 1);
        }
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&kv_empty[i], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS[2] = {tmem, tmem + kBK};
    const uint32_t tO = tmem + 2 * kBK;

    if (warp == 0) {
        // ---------------------------------------------------- TMA producer
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmQ);
            ptx::tma_prefetch_desc(&tmKV);
            int g = 0, it = 0;
            Item I;
            for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
                if (!get_item(p, w, heads, qtiles, I)) continue;
                const int qb = it & 1;
                const int colq = I.head * kD, colk = p.hidden + I.head * kD, colv = 2 * p.hidden + I.head * kD;
                ptx::mbar_wait(&q_empty[qb], ((it >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&q_full[qb], kQBytes);
                ptx::tma_load_2d(&tmQ, &q_full[qb], sQ + qb * kQBytes, colq, I.start + I.q0);
                for (int j = 0; j < I.nblk; ++j, ++g) {
                    const int st = g % kStages;
                    ptx::mbar_wait(&kv_empty[st], ((g / kStages) & 1) ^ 1);
                    ptx::mbar_arrive_expect_tx(&k_full[st], kKVBytes);
                    ptx::tma_load_2d(&tmKV, &k_full[st], sK + st * kKVBytes, colk, I.start + j * kBK);
                    ptx::mbar_arrive_expect_tx(&v_full[st], kKVBytes);
                    ptx::tma_load_2d(&tmKV, &v_full[st], sV + st * kKVBytes, colv, I.start + j * kBK);
                }
                ++it;
            }
            // tail: every ring slot and Q buffer released, i.e. every tcgen05.commit
            // arrive on this CTA's barriers has landed before the CTA can exit
            for (int i = 0; i < kStages; ++i, ++g) ptx::mbar_wait(&kv_empty[g % kStages], ((g / kStages) & 1) ^ 1);
            for (int i = 0; i < 2; ++i, ++it) ptx::mbar_wait(&q_empty[it & 1], ((it >> 1) & 1) ^ 1);
        }
    } else if (warp == 1) {
        // ---------------------------------------------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idS = idesc_f16(kBQ, kBK, 0);
            constexpr uint32_t idO = idesc_f16(kBQ, kD, 1);
            // flattened (item, block) sequence with one S issue of look-ahead
            struct Blk { int g, it, j, nblk; bool valid; };
            int w = blockIdx.x, it = 0, g = 0;
            Item I;
            bool have = false;
            while (w < nitems && !(have = get_item(p, w, heads, qtiles, I))) w += gridDim.x;
            auto first = [&]() { return Blk{g, it, 0, I.nblk, have}; };
            auto advance = [&](const Blk& c) {   // block after c
                if (c.j + 1 < c.nblk) return Blk{c.g + 1, c.it, c.j + 1, c.nblk, true};
                w += gridDim.x;
                have = false;
                while (w < nitems && !(have = get_item(p, w, heads, qtiles, I))) w += gridDim.x;
                return Blk{c.g + 1, c.it + 1, 0, I.nblk, have};
            };
            auto issue_S = [&](const Blk& c) {
                if (c.j == 0) {
                    ptx::mbar_wait(&q_full[c.it & 1], (c.it >> 1) & 1);
                }
                const int st = c.g % kStages;
                ptx::mbar_wait(&k_full[st], (c.g / kStages) & 1);
                ptx::tc_fence_after();
                const uint32_t q_addr = ptx::smem_u32(sQ + (c.it & 1) * kQBytes);
                const uint32_t k_addr = ptx::smem_u32(sK + st * kKVBytes);
#pragma unroll
                for (int k = 0; k < kD / 16; ++k)
                    mma_f16_ss(tS[c.g & 1], ptx::desc_sw128_kmajor(q_addr + 32 * k),
                               ptx::desc_sw128_kmajor(k_addr + 32 * k), idS, k != 0);
                ptx::mma_commit(&s_full[c.g & 1]);
            };
            Blk cur = first();
            if (cur.valid) issue_S(cur);
            while (cur.valid) {
                const Blk nxt = advance(cur);
                if (nxt.valid) issue_S(nxt);
                const int st = cur.g % kStages;
                ptx::mbar_wait(&p_ready[cur.g & 1], (cur.g >> 1) & 1);
                ptx::mbar_wait(&v_full[st], (cur.g / kStages) & 1);
                ptx::tc_fence_after();
                const uint32_t v_addr = ptx::smem_u32(sV + st * kKVBytes);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)   // 16 keys per MMA: 8 TMEM columns of P, 2 KB of V
                    mma_f16_ts(tO, tS[cur.g & 1] + 8 * k, desc_sw128_mnmajor(v_addr + 2048 * k), idO,
                               (cur.j | k) != 0);
                ptx::mma_commit(&kv_empty[st]);
                ptx::mma_commit(&pv_done[cur.g & 1]);
                if (cur.j + 1 == cur.nblk) ptx::mma_commit(&q_empty[cur.it & 1]);
                cur = nxt;
            }
            (void)g;
        }
    } else {
        // ---------------------------------------------------- softmax + epilogue (warps 2-9)
        // warp (q, hf): rows 32q..32q+31 (TMEM lane quadrant q = warp % 4), keys
        // [32hf, 32hf+32) of every block and O dims [32hf, 32hf+32).  The two
        // warps of a quadrant exchange partial row maxima once per block
        // (named barrier 1+q, 64 threads) and partial row sums at the end.
        const int q = warp & 3;
        const int hf = (warp - 2) >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int rl = q * 32 + lane;            // row within the 128-query tile
        const float c = 0.125f * 1.4426950408889634f;   // 1/sqrt(64) * log2(e)
        constexpr int kH = kBK / 2;              // keys per warp per block (32)
        int g = 0;
        Item I;
        for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
            if (!get_item(p, w, heads, qtiles, I)) continue;
            float m = -INFINITY, l = 0.0f;   // reference max (scaled log2 units), row sum w.r.t. m
            for (int j = 0; j < I.nblk; ++j, ++g) {
                ptx::mbar_wait(&s_full[g & 1], (g >> 1) & 1);
                ptx::tc_fence_after();
                uint32_t sv[kH];
                ptx::tmem_ld_32x32b_x32(tS[g & 1] + lane_off + kH * hf, sv);
                ptx::tmem_ld_wait();
                const int kvalid = I.len - j * kBK - kH * hf;   // keys >= kvalid are masked (last block only)
                if (kvalid < kH) {
#pragma unroll
                    for (int i2 = 0; i2 < kH; ++i2)
                        if (i2 >= kvalid) sv[i2] = __float_as_uint(-INFINITY);
                }
                float pm[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) pm[t] = __uint_as_float(sv[t]);
#pragma unroll
                for (int i2 = 8; i2 < kH; ++i2) pm[i2 & 7] = fmaxf(pm[i2 & 7], __uint_as_float(sv[i2]));
                float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                 fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                float* xm = xchg + (g & 1) * 2 * kBQ;
                xm[hf * kBQ + rl] = mx;
                ptx::named_bar_sync(1 + q, 64);
                mx = fmaxf(mx, xm[(hf ^ 1) * kBQ + rl]) * c;   // block max, scaled log2 units
                // lazy rescale: raise the reference only when the block max exceeds it by > 2^8
                const bool up = mx > m + kRescale;
                if (__any_sync(0xffffffffu, up)) {
                    const float m_new = up ? mx : m;
                    const float alpha = ex2f(m - m_new);   // 0 when m = -inf, 1 when !up
                    l *= alpha;
                    if (j > 0) {   // O holds PV_0..PV_{j-1}: wait for PV_{j-1}, then scale our 32 dims
                        ptx::mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
                        ptx::tc_fence_after();
                        uint32_t o[32];
                        ptx::tmem_ld_32x32b_x32(tO + lane_off + 32 * hf, o);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i2 = 0; i2 < 32; ++i2) o[i2] = __float_as_uint(__uint_as_float(o[i2]) * alpha);
                        tmem_st_x32(tO + lane_off + 32 * hf, o);
                    }
                    m = m_new;
                }
                const float nmx = -m;
                float ps[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                uint32_t pk[kH / 2];
#pragma unroll
                for (int i2 = 0; i2 < kH / 2; ++i2) {
                    const float e0 = ex2f(fmaf(__uint_as_float(sv[2 * i2]), c, nmx));
                    const float e1 = ex2f(fmaf(__uint_as_float(sv[2 * i2 + 1]), c, nmx));
                    ps[i2 & 3] += e0 + e1;
                    pk[i2] = h2(e0, e1);
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                // P_j half (fp16, 2 keys per 32-bit column): columns [16hf, 16hf+16)
                tmem_st_x16(tS[g & 1] + lane_off + (kH / 2) * hf, pk);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&p_ready[g & 1]);
                // consume PV_{j-1}'s completion (cheap: it was issued a block ago); keeps
                // every phase of the two pv_done barriers waited on
                if (j > 0) ptx::mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
            }
            // O after the last PV of this item
            ptx::mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
            ptx::tc_fence_after();
            float R[kD / 2];
            {
                uint32_t o[32];
                ptx::tmem_ld_32x32b_x32(tO + lane_off + 32 * hf, o);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i2 = 0; i2 < 32; ++i2) R[i2] = __uint_as_float(o[i2]);
            }
            // ---- epilogue: combine the two halves' row sums, O / l -> quantize -> global
            float* xl = xchg + (g & 1) * 2 * kBQ;   // parity g: not in use by any in-flight block
            xl[hf * kBQ + rl] = l;
            ptx::named_bar_sync(1 + q, 64);
            l += xl[(hf ^ 1) * kBQ + rl];
            ptx::named_bar_sync(1 + q, 64);         // partner has read before the buffer is reused
            const int row = I.q0 + rl;
            if (row < I.len) {
                const float inv = 1.0f / l;
                uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)(I.start + row) * p.ldo;
                const int col0 = I.head * kD + (kD / 2) * hf;   // first output column of this warp
                if (p.out_mode == 0) {
                    float4* dst = reinterpret_cast<float4*>(orow + (int64_t)col0 * 4);
#pragma unroll
                    for (int i2 = 0; i2 < 8; ++i2)
                        dst[i2] = make_float4(R[4 * i2] * inv, R[4 * i2 + 1] * inv, R[4 * i2 + 2] * inv, R[4 * i2 + 3] * inv);
                } else if (p.out_mode == 3) {
                    uint32_t wq[4];
#pragma unroll
                    for (int gq = 0; gq < 4; ++gq) {
                        int qv[8];
#pragma unroll
                        for (int i2 = 0; i2 < 8; ++i2) qv[i2] = quant_code(R[8 * gq + i2] * inv, p.s_out, p.qmin, p.qmax);
                        wq[gq] = pack_nib8(qv);
                    }
                    *reinterpret_cast<uint4*>(orow + col0 / 2) = make_uint4(wq[0], wq[1], wq[2], wq[3]);
                } else {
                    uint32_t wq[8];
#pragma unroll
                    for (int gq = 0; gq < 8; ++gq)
                        wq[gq] = pack_byte4(quant_code(R[4 * gq] * inv, p.s_out, p.qmin, p.qmax),
                                            quant_code(R[4 * gq + 1] * inv, p.s_out, p.qmin, p.qmax),
                                            quant_code(R[4 * gq + 2] * inv, p.s_out, p.qmin, p.qmax),
                                            quant_code(R[4 * gq + 3] * inv, p.s_out, p.qmin, p.qmax));
                    uint4* dst = reinterpret_cast<uint4*>(orow + col0);
                    dst[0] = make_uint4(wq[0], wq[1], wq[2], wq[3]);
                    dst[1] = make_uint4(wq[4], wq[5], wq[6], wq[7]);
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kTmemCols>(tmem);
    }
}

}  // namespace attn2
}  // namespace mkq
