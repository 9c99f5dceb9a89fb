// Microbenchmark (diagnostics): throughput per SMSP of candidate softmax
// instruction mixes on sm_100a -- MUFU ex2 (f32 and f16x2), packed f32x2
// FMA/ADD, three-input max, and a software exp2 (Cody-Waite + degree-3
// polynomial on the FMA pipe, as in FA4) -- to pick the attention exp mix.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/xu_bench2.cu -o build_dbg/xu_bench2
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;"
                 : "=l"(r)
                 : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
                   "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// software 2^x for x <= 0 (FA4-style): j = floor(x), f = x - j in [0,1),
// p(f) ~ 2^f (degree 3), scale by adding j to the exponent field.
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -127.0f);
    const float j = floorf(x);
    const float f = x - j;
    float p = fmaf(fmaf(fmaf(0.0555041086f, f, 0.2402264923f), f, 0.6931471806f), f, 1.0f);
    return __int_as_float(__float_as_int(p) + ((int)j << 23));
}

template <int V>
__global__ void k(int iters, float* out, long long* cyc) {
    float x[16];
    uint32_t acc = 0;
    for (int i = 0; i < 16; ++i) x[i] = -(threadIdx.x * 1e-3f + i * 0.01f);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (V == 0) {   // 2 x MUFU.EX2 f32
                x[i] = ex2f(x[i]);
                x[i + 1] = ex2f(x[i + 1]);
            } else if (V == 1) {   // 1 x ex2.f16x2 (2 values)
                uint32_t h = __float_as_uint(x[i]);
                h = ex2h2(h);
                x[i] = __uint_as_float(h);
            } else if (V == 2) {   // 1 x fma.f32x2 (2 values)
                float2 a = make_float2(x[i], x[i + 1]);
                a = fma2(a, make_float2(0.999f, 0.999f), make_float2(-1e-3f, -1e-3f));
                x[i] = a.x;
                x[i + 1] = a.y;
            } else if (V == 3) {   // 2 x FFMA scalar
                x[i] = fmaf(x[i], 0.999f, -1e-3f);
                x[i + 1] = fmaf(x[i + 1], 0.999f, -1e-3f);
            } else if (V == 4) {   // 1 x 3-input max (2 new values)
                x[0] = max3(x[0], x[i], x[i + 1]);
                x[i] -= 1e-3f;
            } else if (V == 6) {   // 2 x I2FP (cvt.rn.f32.s32)
                x[i] = __int2float_rn(__float_as_int(x[i]) ^ 0x5);
                x[i + 1] = __int2float_rn(__float_as_int(x[i + 1]) ^ 0x5);
            } else if (V == 7) {   // 2 x mad.hi.s32 + add.f32x2 (magic int->float)
                int a0 = __mulhi(__float_as_int(x[i]), 1 << 24) + 0x4B400000;
                int a1 = __mulhi(__float_as_int(x[i + 1]), 1 << 24) + 0x4B400000;
                x[i] = __int_as_float(a0) - 12582912.0f;
                x[i + 1] = __int_as_float(a1) - 12582912.0f;
            } else if (V == 5) {   // 2 x software exp2
                x[i] = ex2_poly(x[i]) - 1.0f;
                x[i + 1] = ex2_poly(x[i + 1]) - 1.0f;
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
    const char* nm[] = {"2x ex2.f32", "1x ex2.f16x2", "1x fma.f32x2", "2x ffma", "1x max3(+1 fadd)", "2x ex2 poly", "2x i2fp(+lop)", "2x mulhi+fadd"};
    for (int warps : {8, 16}) {
        for (int v = 0; v < 8; ++v) {
            const int iters = 2000;
            void (*f)(int, float*, long long*) =
                v == 0 ? k<0> : v == 1 ? k<1> : v == 2 ? k<2> : v == 3 ? k<3> : v == 4 ? k<4> : v == 5 ? k<5> : v == 6 ? k<6> : k<7>;
            f<<<148, 32 * warps>>>(iters, o, c);
            long long h;
            cudaError_t e = cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            const double steps = (double)iters * 8 * (warps / 4);
            printf("warps/SM=%2d %-20s %6.2f cycles per warp pair-step per SMSP\n", warps, nm[v], h / steps);
        }
    }
    return 0;
}
