// Microbenchmark (diagnostics): per-SMSP throughput of the softmax's
// per-element instructions -- MUFU.EX2, F2FP (cvt.rn.f16x2.f32), and the
// integer fp32->fp16 repack -- to see which pipe bounds the exp phase.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/xu_bench.cu -o build_dbg/xu_bench
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
    uint32_t r;
    asm volatile("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
    return r;
}

template <int V>
__global__ void k(int iters, float* out, long long* cyc) {
    float x[16];
    uint32_t acc = 0;
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i * 0.01f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (V == 0) {   // 2 x MUFU.EX2
                x[i] = ex2f(x[i]);
                x[i + 1] = ex2f(x[i + 1]);
            } else if (V == 1) {   // 1 x F2FP
                acc += cvt2(x[i], x[i + 1]);
                x[i] += 1.0f;
            } else if (V == 2) {   // 2 x EX2 + 1 x F2FP
                x[i] = ex2f(x[i]);
                x[i + 1] = ex2f(x[i + 1]);
                acc += cvt2(x[i], x[i + 1]);
            } else {   // 2 x EX2 + integer repack (round-half-up)
                x[i] = ex2f(x[i]);
                x[i + 1] = ex2f(x[i + 1]);
                const uint32_t a = (__float_as_uint(x[i]) + 0x1000u) >> 13;
                const uint32_t b = (__float_as_uint(x[i + 1]) + 0x1000u) << 3;
                acc += a | (b & 0xFFFF0000u);
            }
        }
    }
    const long long t1 = clock64();
    float s = acc;
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    const char* nm[] = {"2x EX2", "1x F2FP", "2x EX2 + F2FP", "2x EX2 + int repack"};
    for (int warps : {4, 8, 16}) {
        for (int v = 0; v < 4; ++v) {
            const int iters = 2000;
            void (*f)(int, float*, long long*) = v == 0 ? k<0> : v == 1 ? k<1> : v == 2 ? k<2> : k<3>;
            f<<<148, 32 * warps>>>(iters, o, c);
            long long h;
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            // per SMSP: warps/4 warps, each iters*8 pair-steps
            const double steps = (double)iters * 8 * (warps / 4);
            printf("warps/SM=%2d %-22s %6.2f cycles per warp-pair-step per SMSP\n", warps, nm[v], h / steps);
        }
    }
    return 0;
}
