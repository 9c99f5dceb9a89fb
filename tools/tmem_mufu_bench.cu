// Microbenchmark (diagnostics): does a warp's tcgen05.ld S readback overlap
// with another warp's MUFU.EX2 work on the same SMSP?  8 warps per CTA, 2 per
// SMSP (warp w on SMSP w & 3): warps 0-3 read 32 TMEM columns x 32 lanes per
// op (ld.x32 + wait), warps 4-7 run ex2.approx on 32 independent values.
// Mode 0: readers only, 1: MUFU only, 2: both, 3: both, MUFU warps also
// pack to f16 (the softmax P path), 4: readers + FFMA2-only warps,
// 5: readers + warps storing 16 TMEM columns per op (st.x16, the P store),
// 6: storers only.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/tmem_mufu_bench.cu -o build_dbg/tmem_mufu_bench
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>

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

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MODE>
__global__ void k(int iters_ld, int iters_mufu, uint32_t* out, long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const bool reader = warp < 4;
    const bool run = MODE == 0 ? reader : ((MODE == 1 || MODE == 6) ? !reader : true);
    uint32_t acc = 0;
    float f[32];
    for (int i = 0; i < 32; ++i) f[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    const long long t0 = clock64();
    if (run && reader) {
        const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t r[32];
        for (int it = 0; it < iters_ld; ++it) {
            ld32(base + 32u * (uint32_t)(it & 7), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r);
        }
    } else if (run && (MODE == 5 || MODE == 6)) {
        // store into the other half of the columns of the same lanes
        const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + 256u;
        uint32_t r[16];
        for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * i;
        for (int it = 0; it < 4 * iters_mufu; ++it) {
            r[0] += 1;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(
                    base + 16u * (uint32_t)(it & 7)),
                "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
            if ((it & 3) == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        acc = r[3];
    } else if (run) {
        for (int it = 0; it < iters_mufu; ++it) {
            if (MODE == 4) {
#pragma unroll
                for (int i = 0; i < 32; ++i) f[i] = fmaf(f[i], 0.999f, 1e-6f);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) f[i] = ex2(f[i]) - 1.0f;
            }
            if (MODE == 3) {
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    __half2 h = __floats2half2_rn(f[i], f[i + 1]);
                    acc ^= *reinterpret_cast<uint32_t*>(&h);
                }
            }
        }
        for (int i = 0; i < 32; ++i) acc ^= __float_as_uint(f[i]);
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) cyc[warp] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    uint32_t* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8 * 8);
    const char* nm[] = {"readers only", "MUFU only", "readers + MUFU", "readers + MUFU+pack", "readers + FFMA",
                        "readers + st.x16", "st.x16 only"};
    void (*fs[])(int, int, uint32_t*, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
    const int il = 4000, im = 1000;
    for (int m = 0; m < 7; ++m) {
        fs[m]<<<148, 256>>>(il, im, o, c);
        long long h[8];
        cudaError_t e = cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        const double rd = (double)h[0], mu = (double)h[4];
        if (m >= 5)
            printf("%-22s reader warp %9.0f cycles (%5.1f B/cycle/SM)   st warp %9.0f cycles (%5.1f B/cycle/SM)\n",
                   nm[m], rd, (m == 6) ? 0.0 : 4.0 * il * 4096 / rd, mu, 4.0 * 4 * im * 2048 / mu);
        else
            printf("%-22s reader warp %9.0f cycles (%5.1f B/cycle/SM)   MUFU warp %9.0f cycles (%.2f cyc per ex2 warp-instr)\n",
                   nm[m], rd, (m == 1) ? 0.0 : 4.0 * il * 4096 / rd, mu, (m == 0) ? 0.0 : mu / (32.0 * im));
    }
    return 0;
}
