// calib.cuh -- SURVEY §8(f) NEXT(4): activation-scale calibration on the GPU
// ("top 0.01% largest value ... as the initial scale", reading R6):
//   a      = |x| sorted ascending (n values)
//   pos    = p (n - 1)  (fp64);  lo = floor(pos);  hi = min(lo + 1, n - 1)
//   quant  = fl32(a[lo] + (pos - lo) (a[hi] - a[lo]))   (fp64 arithmetic)
//   s      = fl32(quant / l_max)
// The order statistics a[lo], a[hi] are found EXACTLY by a radix select on
// the bit patterns of |x| (for non-negative floats the unsigned bit order is
// the numeric order): three histogram passes over 11 + 11 + 9 bits of the
// 31-bit key, each pass counting only the keys whose higher digits match the
// prefix selected so far, one select step after each pass.  Both ranks are
// tracked at once (two prefixes, two histograms per pass).  Nothing is
// sorted and nothing is copied to the host; the index arithmetic (pos, lo,
// hi, frac) is the host's, in the same fp64 operations as the definition.
#pragma once
#include <cstdint>

namespace mkq {
namespace calib {

constexpr int kThreads = 512;
constexpr int kBins = 2048;   // widest digit: 11 bits

struct State {
    unsigned long long k[2];    // rank still to find inside the current prefix
    uint32_t prefix[2];         // selected high bits so far
    uint32_t pad[2];
};
// workspace layout: State | hist[2][kBins] (u64)
constexpr size_t kWsBytes = 64 + 2 * kBins * sizeof(unsigned long long);

__host__ __device__ constexpr int digit_shift(int pass) { return pass == 0 ? 20 : (pass == 1 ? 9 : 0); }
__host__ __device__ constexpr int digit_bits(int pass) { return pass == 2 ? 9 : 11; }

__global__ void init_kernel(State* st, unsigned long long* hist, unsigned long long k_lo, unsigned long long k_hi) {
    for (int i = threadIdx.x; i < 2 * kBins; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
        st->k[0] = k_lo;
        st->k[1] = k_hi;
        st->prefix[0] = st->prefix[1] = 0;
    }
}

// Histogram of digit `pass` over the keys matching each rank's prefix.
template <int kPass>
__global__ void __launch_bounds__(kThreads) hist_kernel(const float* __restrict__ x, int64_t n, int vec,
                                                        const State* __restrict__ st,
                                                        unsigned long long* __restrict__ hist) {
    constexpr int kShift = digit_shift(kPass), kDb = digit_bits(kPass), kNb = 1 << kDb;
    constexpr uint32_t kHiMask = kPass == 0 ? 0u : (0x7FFFFFFFu >> (kShift + kDb)) << (kShift + kDb);
    __shared__ uint32_t h[2][kNb];
    for (int i = threadIdx.x; i < 2 * kNb; i += blockDim.x) (&h[0][0])[i] = 0;
    const uint32_t p0 = st->prefix[0], p1 = st->prefix[1];
    const bool same = p0 == p1;
    __syncthreads();
    auto add = [&](float v) {
        const uint32_t u = __float_as_uint(v) & 0x7FFFFFFFu;
        const uint32_t d = (u >> kShift) & (kNb - 1);
        const uint32_t hb = u & kHiMask;
        if (hb == p0) atomicAdd(&h[0][d], 1u);
        if (!same && hb == p1) atomicAdd(&h[1][d], 1u);
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (vec) {
        const int64_t n4 = n >> 2;
        const float4* x4 = reinterpret_cast<const float4*>(x);
        int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {   // 4 x 16 B in flight per thread
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(x4 + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) { add(v[u].x); add(v[u].y); add(v[u].z); add(v[u].w); }
        }
        for (; i < n4; i += stride) {
            const float4 v = __ldg(x4 + i);
            add(v.x); add(v.y); add(v.z); add(v.w);
        }
        for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) add(x[i]);
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) add(x[i]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kNb; i += blockDim.x) {
        if (h[0][i]) atomicAdd(hist + i, (unsigned long long)h[0][i]);
        if (h[1][i]) atomicAdd(hist + kBins + i, (unsigned long long)h[1][i]);
    }
}

// Select step (one block): for each rank, find the bin b with
// cum(b) <= k < cum(b) + count(b); append b to the prefix, k -= cum(b);
// clear the histograms for the next pass.
template <int kPass>
__global__ void __launch_bounds__(kThreads) select_kernel(State* __restrict__ st, unsigned long long* __restrict__ hist) {
    constexpr int kShift = digit_shift(kPass), kNb = 1 << digit_bits(kPass);
    constexpr int kPer = kNb / kThreads;   // 4 (11-bit) or 1 (9-bit)
    __shared__ unsigned long long wsum[kThreads / 32];
    const bool same = st->prefix[0] == st->prefix[1];
    for (int r = 0; r < 2; ++r) {
        const unsigned long long* hr = hist + (same ? 0 : r) * kBins;
        const unsigned long long k = st->k[r];
        unsigned long long c[kPer], tot = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) { c[j] = hr[threadIdx.x * kPer + j]; tot += c[j]; }
        // block exclusive scan of tot
        unsigned long long incl = tot;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        unsigned long long base = 0;
        for (int i = 0; i < w; ++i) base += wsum[i];
        unsigned long long cum = base + incl - tot;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (c[j] && cum <= k && k < cum + c[j]) {
                st->prefix[r] |= (uint32_t)(threadIdx.x * kPer + j) << kShift;
                st->k[r] = k - cum;
            }
            cum += c[j];
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < 2 * kBins; i += blockDim.x) hist[i] = 0;
}

// quant = fl32(a_lo + frac (a_hi - a_lo)) in fp64 (no contraction);
// s = fl32(quant / l_max).
__global__ void finalize_kernel(const State* __restrict__ st, double frac, float l_max, float* __restrict__ s_out) {
    const double a_lo = (double)__uint_as_float(st->prefix[0]);
    const double a_hi = (double)__uint_as_float(st->prefix[1]);
    const float q = __double2float_rn(__dadd_rn(a_lo, __dmul_rn(frac, __dsub_rn(a_hi, a_lo))));
    s_out[0] = __fdiv_rn(q, l_max);
}

}  // namespace calib
}  // namespace mkq
