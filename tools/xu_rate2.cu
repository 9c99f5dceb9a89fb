// Microbenchmark (diagnostics): per-SMSP issue cost of the half-precision MUFU
// exponentials (ex2.approx.f16x2 / bf16x2) against ex2.approx.f32, the 3-input
// max.f32 (sm_100), HADD2 and f16 -> f32 conversion, on sm_100a.  Build:
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/xu_rate2.cu -o build_dbg/xu_rate2
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
template <int MODE>
__global__ void k(int iters, float* out, long long* cyc) {
    uint32_t a[8];
    float f[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = threadIdx.x * 1e-3f + i * 0.01f - 1.0f;
        __half2 h = __floats2half2_rn(f[i], f[i] * 0.5f);
        a[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
            } else if (MODE == 1) {
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
            } else if (MODE == 2) {
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
            } else if (MODE == 3) {
                asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
            } else if (MODE == 4) {
                asm volatile("max.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]));
            } else if (MODE == 5) {
                asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i + 1) & 7]));
            } else if (MODE == 6) {
                float lo;
                asm volatile("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f32.f16 %0, l;}" : "=f"(lo) : "r"(a[i]));
                f[i] += lo;
            } else if (MODE == 7) {   // f32x2 -> f16x2 pack then f16x2 ex2 (the proposed softmax step)
                uint32_t r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[i]), "f"(f[(i + 1) & 7]));
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r));
                f[i] = __uint_as_float(__float_as_uint(f[i]) ^ (r & 0x80000000u));
            } else if (MODE == 8) {   // mixed-precision add f32 += f16 (sm_100)
                asm volatile("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, l, %0;}" : "+f"(f[i]) : "r"(a[i]));
            }
        }
    }
    const long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(a[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    const char* nm[] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2", "max.f32 (3 inputs)",
                        "max.f32 (2 inputs)", "add.rn.f16x2", "cvt.f32.f16", "cvt.f16x2 + ex2.f16x2",
                        "add.rn.f32.f16"};
    void (*fs[])(int, float*, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>};
    for (int warps : {4, 8, 16}) {
        for (int m = 0; m < 9; ++m) {
            const int iters = 2000;
            fs[m]<<<148, 32 * warps>>>(iters, o, c);
            long long hc;
            cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)iters * 8 * warps;
            printf("warps=%2d %-24s %6.2f warp-inst/cycle/SM (%.2f cycles per warp-inst per SMSP)\n", warps, nm[m],
                   ops / hc, 4.0 * hc / ops);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
