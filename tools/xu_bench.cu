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

// The attention kernel's exp loop on 128 register values per thread (one
// query row x 128 keys): FFMA + MUFU.EX2 + FADD + F2FP, optionally with the
// tcgen05.st of P (V=1).
template <int V>
__global__ void softmax_loop(int iters, float* out, long long* cyc) {
    __shared__ uint32_t slot;
    if (V) {
        if (threadIdx.x < 32) asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    const uint32_t taddr = V ? slot + ((uint32_t)((threadIdx.x >> 5) & 3) * 32 << 16) : 0;
    float sv[128];
    for (int i = 0; i < 128; ++i) sv[i] = (threadIdx.x * 7 + i * 13) % 31 * 0.1f;
    float l = 0.f;
    const float c = 0.18033687f;
    float nmx = -2.0f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float e0 = ex2f(fmaf(sv[32 * cc + 2 * i], c, nmx));
                const float e1 = ex2f(fmaf(sv[32 * cc + 2 * i + 1], c, nmx));
                ps[i & 3] += e0 + e1;
                pk[i] = cvt2(e0, e1);
            }
            if (V) {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                    "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr + 16 * cc),
                    "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]), "r"(pk[8]),
                    "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]), "r"(pk[14]), "r"(pk[15])
                    : "memory");
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) l += __uint_as_float(pk[i]) * 1e-30f;
            }
        }
        if (V) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
        nmx = -2.0f - (float)(it & 3) * 1e-3f;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = l;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    if (V) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
    }
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
    for (int warps : {4, 8}) {
        for (int v = 0; v < 2; ++v) {
            const int iters = 200;
            (v ? softmax_loop<1> : softmax_loop<0>)<<<148, 32 * warps>>>(iters, o, c);
            long long h;
            cudaError_t e = cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            printf("warps/SM=%2d softmax exp loop %s: %7.1f cycles per 128-key row block (MUFU floor %d)\n", warps,
                   v ? "with tcgen05.st" : "registers only ", (double)h / iters, 1024 * warps / 4);
        }
    }
    return 0;
}
