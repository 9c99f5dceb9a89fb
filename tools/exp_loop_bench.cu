// Microbenchmark (diagnostics): the attention softmax's per-block exp phase
// (attention_pp_sm100.cuh: 128 scores per thread -> x = s*c - m (FFMA2) ->
// 2^x (MUFU, or the FMA-pipe polynomial for pairs (i & 7) >= kPolyFrom) ->
// row sum (FADD2) -> fp16 pack -> tcgen05.st of P), timed per warp with
// clock64.  Modes: 0 one exp warp per SMSP, 1 two exp warps per SMSP,
// 2 one exp warp + one TMEM-reader warp per SMSP (the ping-pong pairing).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2203_13483_b200/csrc tools/exp_loop_bench.cu
#include <cstdint>
#include <cstdio>
#include "attention_sm100.cuh"

using namespace mkq::attn2;
#ifndef VARIANT
#define VARIANT "full"
#endif
#ifndef POLY_FROM
#define POLY_FROM 6
#endif

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// folds all 32 results (a dynamically indexed r[it & 31] would put the array
// in local memory and time the local stores instead of the TMEM reads; an
// empty asm "use" lets ptxas delete the unused loads)
__device__ __forceinline__ uint32_t fold(const uint32_t (&r)[32]) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= r[i];   // 3-input LOP3s: ~16 ALU ops per 32 registers
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int iters, uint32_t* out, long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16);
    const bool expw = warp < 4 || MODE == 1;
    const bool active = warp < 4 || MODE != 0;
    uint32_t acc = 0;
    const float c = 0.125f * 1.4426950408889634f;
    uint32_t sv[4][32];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[cc][i] = __float_as_uint(-0.01f * (float)((lane * 7 + i * 3 + cc * 5) & 63));
    float l = 0.0f;
    __syncthreads();
    const long long t0 = clock64();
    if (active && expw) {
        const uint32_t tP = tm + 384u + (warp >= 4 ? 64u : 0u);
        for (int it = 0; it < iters; ++it) {
            const float nmx = -0.25f * (float)(it & 3);
            float2 ps2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
#ifdef SCALAR
                    const float2 x2 = make_float2(fmaf(__uint_as_float(sv[cc][2 * i]), c, nmx),
                                                  fmaf(__uint_as_float(sv[cc][2 * i + 1]), c, nmx));
#else
                    const float2 x2 = ffma2(make_float2(__uint_as_float(sv[cc][2 * i]), __uint_as_float(sv[cc][2 * i + 1])),
                                            make_float2(c, c), make_float2(nmx, nmx));
#endif
                    const float2 e2 = (i & 7) >= POLY_FROM ? ex2_fma2(x2) : make_float2(ex2f(x2.x), ex2f(x2.y));
#ifndef NOSUM
#ifdef SCALAR
                    ps2[i & 1].x += e2.x;
                    ps2[i & 1].y += e2.y;
#else
                    ps2[i & 1] = fadd2(ps2[i & 1], e2);
#endif
#endif
#ifdef NOPACK
                    pk[i] = __float_as_uint(e2.x) ^ __float_as_uint(e2.y);
#else
                    pk[i] = h2(e2.x, e2.y);
#endif
                }
#ifdef NOST
#pragma unroll
                for (int i = 0; i < 16; ++i) acc ^= pk[i];
#else
                tmem_st_x16(tP + 16 * cc, pk);
#endif
            }
            l += (ps2[0].x + ps2[1].x) + (ps2[0].y + ps2[1].y);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        acc ^= __float_as_uint(l);
    } else if (active) {
        uint32_t r[32];
        for (int it = 0; it < 4 * iters; ++it) {
            ld32(tm + 32u * (uint32_t)(it & 3), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r);
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (blockIdx.x == 0 && lane == 0) cyc[warp] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    uint32_t* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8 * 8);
    const char* nm[] = {"1 exp warp / SMSP", "2 exp warps / SMSP", "1 exp + 1 reader / SMSP"};
    void (*fs[])(int, uint32_t*, long long*) = {k<0>, k<1>, k<2>};
    const int iters = 2000;
    for (int m = 0; m < 3; ++m) {
        fs[m]<<<148, 256>>>(iters, o, c);
        long long h[8];
        cudaError_t e = cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("%-24s POLY_FROM=%d %-26s exp warp: %6.0f cycles per 128-key block (4096 exps)   warp4: %6.0f\n", VARIANT, POLY_FROM,
               nm[m], (double)h[0] / iters, (double)h[4] / iters);
    }
    return 0;
}
