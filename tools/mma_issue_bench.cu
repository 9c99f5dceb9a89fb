// Microbenchmark (diagnostics): issue and completion cost of back-to-back
// tcgen05.mma kind::f16 instructions from one thread, as used by the
// attention kernel (SS 128x128x16 for S = Q K^T, TS 128x64x16 for O += P V).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2203_13483_b200/csrc -I include tools/mma_issue_bench.cu -o build_dbg/mma_bench
#include <cstdio>
#include <cuda.h>
#include <cuda_fp16.h>
#include "attention_sm100.cuh"

using namespace mkq;

__device__ __forceinline__ void mma_f16_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_f16_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__global__ void bench(int variant, int nmma, int reps, int busy, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    ptx::fence_proxy_async_smem();
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0) {
        if (lane == 0 && variant < 3) {
            const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
            const uint32_t idS = attn2::idesc_f16(128, 128, 0), idO = attn2::idesc_f16(128, 64, 1);
            unsigned long long t_issue = 0, t_done = 0;
            for (int r = 0; r < reps; ++r) {
                const unsigned long long t0 = clock64();
                for (int k = 0; k < nmma; ++k) {
                    if (variant == 0)
                        attn2::mma_f16_ss(tmem, ptx::desc_sw128_kmajor(a + 32 * (k & 3)),
                                          ptx::desc_sw128_kmajor(b + 32 * (k & 3)), idS, k != 0);
                    else if (variant == 1)
                        attn2::mma_f16_ts(tmem + 256, tmem + 384 + 8 * (k & 7),
                                          attn2::desc_sw128_mnmajor(b + 2048 * (k & 7)), idO, k != 0);
                    else
                        attn2::mma_f16_ss(tmem + 256, ptx::desc_sw128_kmajor(a + 32 * (k & 3)),
                                          attn2::desc_sw128_mnmajor(b + 2048 * (k & 7)), idO, k != 0);
                }
                const unsigned long long t1 = clock64();
                ptx::mma_commit(&bar);
                ptx::mbar_wait(&bar, r & 1);
                const unsigned long long t2 = clock64();
                t_issue += t1 - t0;
                t_done += t2 - t0;
            }
            out[0] = t_issue;
            out[1] = t_done;
        }
        if (variant >= 3) {   // whole warp converged, elect.sync inside the asm
            const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
            const uint32_t idS = attn2::idesc_f16(128, 128, 0), idO = attn2::idesc_f16(128, 64, 1);
            unsigned long long t_issue = 0, t_done = 0;
            const uint64_t da = ptx::desc_sw128_kmajor(a), db = ptx::desc_sw128_kmajor(b);
            const uint64_t dv = attn2::desc_sw128_mnmajor(b);
            for (int r = 0; r < reps; ++r) {
                __syncwarp();
                const unsigned long long t0 = clock64();
                if (variant == 3) {
#pragma unroll 8
                    for (int k = 0; k < nmma; ++k)
                        mma_f16_ts_elect(tmem + 256, tmem + 384 + 8 * (k & 7), dv + 128 * (k & 7), idO, k != 0);
                } else {
#pragma unroll 4
                    for (int k = 0; k < nmma; ++k)
                        mma_f16_ss_elect(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idS, k != 0);
                }
                __syncwarp();
                const unsigned long long t1 = clock64();
                if (lane == 0) ptx::mma_commit(&bar);
                ptx::mbar_wait(&bar, r & 1);
                const unsigned long long t2 = clock64();
                t_issue += t1 - t0;
                t_done += t2 - t0;
            }
            if (lane == 0) {
                out[0] = t_issue;
                out[1] = t_done;
            }
        }
    } else if (busy) {
        // MUFU-heavy busy warps (like the softmax), until warp 0 is done
        float x = threadIdx.x * 1e-3f;
        for (int i = 0; i < busy; ++i) {
#pragma unroll 16
            for (int k = 0; k < 64; ++k) x = attn2::ex2f(x * 0.999f - 0.5f);
        }
        if (x == 12345.f) out[2] = 1;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// Exp-loop throughput of 4 warps (one per SMSP) while warp 0 keeps the
// tensor core busy with MMAs (mode 1: SS 128x128x16, 2: TS 128x64x16) or idle (0).
__global__ void exp_vs_mma(int mode, int iters, float* fout, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
        done = 0;
    }
    ptx::fence_proxy_async_smem();
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0) {
        if (mode) {
            const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
            const uint64_t da = ptx::desc_sw128_kmajor(a), db = ptx::desc_sw128_kmajor(b);
            const uint64_t dv = attn2::desc_sw128_mnmajor(b);
            const uint32_t idS = attn2::idesc_f16(128, 128, 0), idO = attn2::idesc_f16(128, 64, 1);
            int r = 0;
            while (!done) {
                for (int k = 0; k < 16; ++k) {
                    if (mode == 1) attn2::mma_f16_ss_warp(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idS, k != 0);
                    else attn2::mma_f16_ts_warp(tmem + 256, tmem + 384 + 8 * (k & 7), dv + 128 * (k & 7), idO, k != 0);
                }
                ptx::mma_commit_warp(&bar);
                ptx::mbar_wait(&bar, r & 1);
                ++r;
            }
        }
    } else {
        float sv[128];
        for (int i = 0; i < 128; ++i) sv[i] = ((threadIdx.x * 7 + i * 13) % 61) * -0.5f;
        float l = 0.f;
        const float c = 0.18033687f;
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const float nmx = -2.0f - (float)(it & 3) * 1e-3f;
            float ps[4] = {0.f, 0.f, 0.f, 0.f};
            uint32_t acc = 0;
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                const float e0 = attn2::ex2f(fmaf(sv[2 * i], c, nmx));
                const float e1 = attn2::ex2f(fmaf(sv[2 * i + 1], c, nmx));
                ps[i & 3] += e0 + e1;
                acc ^= attn2::h2(e0, e1);
            }
            l += (ps[0] + ps[1]) + (ps[2] + ps[3]) + (float)(acc & 1);
        }
        const unsigned long long t1 = clock64();
        fout[threadIdx.x] = l;
        if (threadIdx.x == 32) out[0] = t1 - t0;
        __syncwarp();
        if (threadIdx.x == 32) done = 1;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    const char* names[] = {"SS 128x128x16 (S=QK^T)", "TS 128x64x16 (O+=PV)", "SS 128x64x16 (MN-major B)",
                           "TS 128x64x16 warp+elect", "SS 128x128x16 warp+elect"};
    for (int busy = 0; busy <= 1; ++busy)
        for (int v = 0; v < 5; ++v)
            for (int n : {4, 8, 16, 64}) {
                const int reps = 50;
                bench<<<1, busy ? 320 : 32, 70000>>>(v, n, reps, busy ? 4000 : 0, d);
                unsigned long long h[2];
                cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                printf("%-28s busy=%d n=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma\n", names[v], busy, n,
                       (double)h[0] / reps / n, (double)h[1] / reps / n);
            }
    float* fo;
    cudaMalloc(&fo, 4096);
    cudaFuncSetAttribute(exp_vs_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    const char* mn[] = {"tensor idle", "SS 128x128x16 stream", "TS 128x64x16 stream"};
    for (int mode = 0; mode < 3; ++mode) {
        const int iters = 200;
        exp_vs_mma<<<1, 160, 70000>>>(mode, iters, fo, d);
        unsigned long long h;
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        printf("exp loop (128 exps/thread, 1 warp/SMSP) with %-22s: %7.1f cycles per block (MUFU floor 1024)\n", mn[mode],
               (double)h / iters);
    }
    return 0;
}
