// Microbenchmark (diagnostics): tcgen05.ld / tcgen05.st throughput per SM on
// sm_100a, for the attention softmax's S readback (32x32b.x32 per warp).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/tmem_bench.cu -o build_dbg/tmem_bench
#include <cstdint>
#include <cstdio>

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
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void ld16x256_x8(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void ld16x128_x16(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x128b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// 0: ld + wait each (same columns every iteration), 1: 4 lds then wait (columns ^64/128/192),
// 2: st x32 (+wait::st every 4), 3: 16x256b.x8, 4: 16x128b.x16,
// 5: ld + wait, columns rotating over 8 x 32 (distinct data each time),
// 6: 4 lds of consecutive 32-column chunks then wait (the attention S readback pattern),
// 7: 2 lds (consecutive chunks) then wait
template <int MODE>
__global__ void k(int iters, uint32_t* out, long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32 % 512);
    uint32_t acc = 0;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            ld32(base, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r);
        } else if (MODE == 1) {
            uint32_t a[32], b[32], c[32];
            ld32(base, r);
            ld32(base ^ 64, a);
            ld32(base ^ 128, b);
            ld32(base ^ 192, c);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r) ^ fold(a) ^ fold(b) ^ fold(c);
        } else if (MODE == 5) {
            ld32(base + 32u * (uint32_t)((it + (warp >> 2)) & 7), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r);
        } else if (MODE == 6) {
            uint32_t a[32], b[32], c[32];
            const uint32_t b0 = slot + ((uint32_t)((warp & 3) * 32) << 16) + 128u * (uint32_t)((it + (warp >> 2)) & 3);
            ld32(b0, r);
            ld32(b0 + 32, a);
            ld32(b0 + 64, b);
            ld32(b0 + 96, c);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r) ^ fold(a) ^ fold(b) ^ fold(c);
        } else if (MODE == 7) {
            uint32_t a[32];
            const uint32_t b0 = slot + ((uint32_t)((warp & 3) * 32) << 16) + 64u * (uint32_t)((it + (warp >> 2)) & 7);
            ld32(b0, r);
            ld32(b0 + 32, a);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r) ^ fold(a);
        } else if (MODE == 3) {
            ld16x256_x8(base, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r);
        } else if (MODE == 4) {
            ld16x128_x16(base, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= fold(r);
        } else {
            r[0] += 1;   // static index: r stays in registers
            st32(base, r);
            if ((it & 3) == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    uint32_t* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    const char* nm[] = {"ld.x32 + wait", "4 x ld.x32 + wait", "st.x32", "16x256b.x8 + wait", "16x128b.x16 + wait",
                        "ld.x32 rotating", "4 x ld.x32 consec", "2 x ld.x32 consec"};
    void (*fs[])(int, uint32_t*, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>};
    const int mult[] = {1, 4, 1, 1, 1, 1, 4, 2};
    for (int warps : {4, 8, 16}) {
        for (int m = 0; m < 8; ++m) {
            const int iters = 4000;
            void (*f)(int, uint32_t*, long long*) = fs[m];
            f<<<148, 32 * warps>>>(iters, o, c);
            long long h;
            cudaError_t e = cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            const double bytes = (double)iters * warps * 4096 * mult[m];
            printf("warps=%2d %-18s %7.1f B/cycle/SM (%.0f cycles per op per warp)\n", warps, nm[m], bytes / h,
                   (double)h / iters / mult[m]);
        }
    }
    return 0;
}
