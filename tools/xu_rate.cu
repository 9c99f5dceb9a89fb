// Microbenchmark (diagnostics): per-SM throughput of MUFU.EX2, F2FP (f32x2 -> f16x2
// pack), their mix, and FFMA2, on sm_100a.  Build:
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/xu_rate.cu -o build_dbg/xu_rate
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
template <int MODE>
__global__ void k(int iters, float* out, long long* cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 0.01f;
    uint32_t h = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {   // ex2
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            } else if (MODE == 1) {   // f2fp pack
                uint32_t r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                h ^= r;
                a[i] = __uint_as_float(__float_as_uint(a[i]) ^ r);
            } else if (MODE == 2) {   // ffma2
                uint64_t r;
                asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(r) : "l"(*reinterpret_cast<uint64_t*>(&a[i & 6])));
                *reinterpret_cast<uint64_t*>(&a[i & 6]) = r;
            } else {   // 1 ex2 + 1/2 f2fp per element (the softmax mix)
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                if (i & 1) {
                    uint32_t r;
                    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i - 1]));
                    h ^= r;
                }
            }
        }
    }
    const long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + h;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    const char* nm[] = {"ex2.approx.f32", "cvt.rn.f16x2.f32", "fma.rn.f32x2", "ex2 + 1/2 cvt"};
    void (*fs[])(int, float*, long long*) = {k<0>, k<1>, k<2>, k<3>};
    for (int warps : {4, 8, 16}) {
        for (int m = 0; m < 4; ++m) {
            const int iters = 2000;
            fs[m]<<<148, 32 * warps>>>(iters, o, c);
            long long hc;
            cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)iters * 8 * warps;   // warp-instructions of the measured op per SM
            printf("warps=%2d %-18s %6.2f warp-inst/cycle/SM (%.1f cycles per warp-inst per SMSP)\n", warps, nm[m],
                   ops / hc, 4.0 * hc / ops);
        }
    }
    return 0;
}
