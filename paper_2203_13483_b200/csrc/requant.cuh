// requant.cuh -- exact lookup table for the fused GELU + requantize epilogue
// (§8a rows a5-a6; SURVEY §7.3-3 "epilogue ALU budget").
//
// The FFN1 epilogue maps y = fma((float)acc, sc[n], b[n]) to the FFN2 input
// code  c(y) = clamp(rint_even(gelu_pinned(y) / s_out), qmin, qmax)  (R2-R7).
// c depends on the fp32 value y only -- not on the column -- so one table in
// y-space serves every column.  Evaluating gelu_pinned + an IEEE division per
// output costs ~45 ALU ops, more than the tensor core leaves per output at
// K = 1024; the table replaces them by a cell index, one shared-memory load
// and one compare:
//     cell i = clamp(floor(fma(y, inv_w, c0)))          (same fp32 ops as here)
//     c      = y >= thr[i] ? above[i] : below[i]       (exact fp32 compare)
// Exactness is by construction, not by approximation: the builder evaluates
// c(y) with the SAME device functions for EVERY fp32 y where c can change
// (all floats in [y_lo, -y_zero] and [y_zero, y_hi]); outside those ranges c
// is constant by proof (|gelu_pinned(y)| <= |y| gives c = 0 for |y| < 0.49 s;
// gelu_pinned(y) = 0 for y <= -5.6 and = y for y >= 5.6).  A cell holding more
// than one change point is flagged `direct` and evaluated with the full
// pipeline.  A verify pass re-checks lookup == direct for every float of the
// scanned ranges and clears `valid` on any mismatch (the epilogue then falls
// back to direct evaluation); nothing here needs a host synchronization.
#pragma once
#include <cstdint>
#include "epilogue.cuh"

namespace mkq {
namespace rq {

constexpr int kCells = 1024;
constexpr int kMaxChanges = 4096;

struct Header {
    float c0, y_hi, inv_w, y_zero;   // c0 = fl(-y_lo * inv_w)
    int ncell, code_lo, code_hi, valid;
    int gelu, qmin, qmax, nchg;
    float s_out;
    float y_lo;
    int pad[2];
};   // 64 bytes

struct Change {
    float y;
    int before, after, pad;
};

// ---- compact int4 table (the FFN1 epilogue's fast path; int4 outputs only)
// 256 cells over the span of the change points, one 32-bit word per cell:
//     cell(y) = RN(255 * sat(fma(y, a, b)))  in [0, 255]   (cell4 below)
//     word    = (F - 256) | below | above << 4                      (>= 1 change)
//             = 0x7F800000 | below | below << 4  (NaN: y >= it is false)  (none)
// where every change point of the cell lies in the 256-float run
// R = {bits in [F, F + 256)}, F a multiple of 256.  The word sits just below
// R (in magnitude), so the window  D = {bits(y) - word < kWin4}  (unsigned,
// kWin4 = 512: bits in [word, word + 512) >= [F - 1, F + 256)) contains R, and
// outside D the fp32 compare  y >= float(word)  decides exactly (above R or
// below R, for either sign of the threshold).  The epilogue computes
// bits(y) - word with one IMAD (FMA pipe) and evaluates the lanes in D
// directly.  A cell whose change points do not fit one R makes the table
// invalid.  In shared
// memory each word is replicated 32 times (lane l reads bank l), so a warp's
// 32 lookups are one conflict-free wavefront.
constexpr int kCells4 = 256;
struct Header4 {
    float a, b;
    int valid, pad[13];
};   // 64 bytes

// table bytes: header + cells (uint2: thr bits, meta) + header4 + cells4 + change scratch
constexpr size_t kOff4 = sizeof(Header) + kCells * 8;
constexpr size_t kTableBytes = kOff4 + sizeof(Header4) + kCells4 * 4 + kMaxChanges * sizeof(Change);
constexpr size_t kSmemBytes = sizeof(Header) + kCells * 8;
constexpr size_t kSmem4Bytes = kCells4 * 32 * 4;   // replicated cells4

__device__ __forceinline__ float fma_sat(float x, float a, float b) {
    float r;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x), "f"(a), "f"(b));
    return r;
}
// cell of the compact table, the epilogue's exact sequence: u = sat(fma(y, a, b))
// in [0, 1], then fma(u, 255, 2^23) lies in [2^23, 2^23 + 255] where the ulp is
// 1, so its mantissa is the cell RN(255 u) (no float->int conversion).
constexpr uint32_t kMagic = 0x4B000000u;   // bits of 2^23
__device__ __forceinline__ uint32_t cell4(float y, float a, float b) {
    return __float_as_uint(__fmaf_rn(fma_sat(y, a, b), 255.0f, 8388608.0f)) - kMagic;
}
// 0 = decided: *code = the int4 field; 1 = y is in the cell's direct-
// evaluation window D (the kWin4 floats from the threshold word up in magnitude)
constexpr uint32_t kWin4 = 512u;
__device__ __forceinline__ bool lookup4(uint32_t w, float y, uint32_t* field) {
    if (__float_as_uint(y) - w < kWin4) return true;
    *field = (y >= __uint_as_float(w) ? (w >> 4) : w) & 0xFu;
    return false;
}

__device__ __forceinline__ int direct_code(float y, int gelu, float s, int qmin, int qmax) {
    return quant_code(gelu ? gelu_pinned(y) : y, s, qmin, qmax);
}

// cell index: floor(fma(y, inv_w, c0)) clamped; monotone non-decreasing in y
// (RN of a monotone real function), identical on the build and lookup sides.
__device__ __forceinline__ int cell_of(float y, float c0, float inv_w, int ncell) {
    int i = __float2int_rd(__fmaf_rn(y, inv_w, c0));
    return min(max(i, 0), ncell - 1);
}

// meta: byte 0 code_below, byte 1 code_above, bit 16 direct.  Codes are
// stored as the output's packed field: a 4-bit nibble (0..15, the int4 two's
// complement) for int4 tables (qmin >= -8, qmax <= 7), a byte otherwise, so
// the epilogue selects one with a single PRMT and packs without masking.
__device__ __forceinline__ bool is_int4(int qmin, int qmax) { return qmin >= -8 && qmax <= 7; }

__device__ __forceinline__ int decode_field(uint32_t f, bool int4) {
    return int4 ? (int)(f & 0xF) - (int)((f & 0x8) << 1) : (int)(int8_t)(f & 0xFF);
}

// cell index with an unsigned saturating conversion (negatives -> 0) and one
// min: the epilogue's exact sequence
__device__ __forceinline__ uint32_t cell_u(float y, float c0, float inv_w, uint32_t ncell) {
    uint32_t i;
    asm("cvt.rmi.u32.f32 %0, %1;" : "=r"(i) : "f"(__fmaf_rn(y, inv_w, c0)));
    return min(i, ncell - 1u);
}

// Exactly the epilogue's lookup: no range tests -- cells clamp, cell 0's
// "below" is code_lo and every cell past the last change point holds code_hi.
__device__ __forceinline__ int lookup(const Header& h, const uint2* cells, float y) {
    const uint2 e = cells[cell_u(y, h.c0, h.inv_w, (uint32_t)h.ncell)];
    if (e.y & 0x10000u) return direct_code(y, h.gelu, h.s_out, h.qmin, h.qmax);
    const uint32_t f = __byte_perm(e.y, 0, y >= __uint_as_float(e.x) ? 0x4441 : 0x4440);
    return decode_field(f, is_int4(h.qmin, h.qmax));
}

__device__ __forceinline__ float next_down(float y) {   // largest float < y (y finite, != -0)
    const uint32_t b = __float_as_uint(y);
    if (y > 0.0f) return __uint_as_float(b - 1);
    if (y == 0.0f) return -__uint_as_float(1u);
    return __uint_as_float(b + 1);
}

// Range r in {0: positive [y_zero, y_hi], 1: negative [y_lo, -y_zero]} as a
// run of consecutive floats in increasing y order: index k -> y.
__device__ __forceinline__ float range_y(int r, uint32_t b0, uint32_t n, uint32_t k) {
    // positive: bits b0..b0+n-1 ascending; negative: magnitudes from the top down
    return r == 0 ? __uint_as_float(b0 + k) : -__uint_as_float(b0 + (n - 1 - k));
}

__global__ void scan_kernel(Header* h, Change* chg, uint32_t bp0, uint32_t np, uint32_t bn0, uint32_t nn) {
    const uint32_t total = np + nn;
    constexpr uint32_t kRun = 64;
    const uint32_t runs = (total + kRun - 1) / kRun;
    const int gelu = h->gelu, qmin = h->qmin, qmax = h->qmax;
    const float s = h->s_out;
    for (uint32_t run = blockIdx.x * blockDim.x + threadIdx.x; run < runs; run += gridDim.x * blockDim.x) {
        const uint32_t k0 = run * kRun;
        const uint32_t k1 = min(k0 + kRun, total);
        // runs never straddle the two ranges: split at np
        uint32_t k = k0;
        while (k < k1) {
            const int r = k < np ? 0 : 1;
            const uint32_t kend = r == 0 ? min(k1, np) : k1;
            const uint32_t b0 = r == 0 ? bp0 : bn0, n = r == 0 ? np : nn, kk0 = r == 0 ? k : k - np;
            float y = range_y(r, b0, n, kk0);
            int prev = direct_code(next_down(y), gelu, s, qmin, qmax);
            for (uint32_t kk = kk0; kk < kk0 + (kend - k); ++kk) {
                y = range_y(r, b0, n, kk);
                const int c = direct_code(y, gelu, s, qmin, qmax);
                if (c != prev) {
                    const int i = atomicAdd(&h->nchg, 1);
                    if (i < kMaxChanges) chg[i] = Change{y, prev, c, 0};
                }
                prev = c;
            }
            k = kend;
        }
    }
}

__device__ __forceinline__ uint32_t ord_key(float y) {   // monotone float -> uint
    const uint32_t b = __float_as_uint(y);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void finalize_kernel(Header* h, uint2* cells, Change* chg) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int n = h->nchg;
    if (n > kMaxChanges) { h->valid = 0; return; }
    for (int i = 1; i < n; ++i) {   // insertion sort by y (n is small: <= ~300)
        Change c = chg[i];
        int j = i - 1;
        while (j >= 0 && ord_key(chg[j].y) > ord_key(c.y)) { chg[j + 1] = chg[j]; --j; }
        chg[j + 1] = c;
    }
    int run = h->code_lo;
    int p = 0;
    bool ok = true;
    for (int i = 0; i < h->ncell; ++i) {
        int cnt = 0;
        float thr = 0.0f;
        int below = run, above = run;
        while (p < n && (int)cell_u(chg[p].y, h->c0, h->inv_w, (uint32_t)h->ncell) == i) {
            if (cnt == 0) { thr = chg[p].y; if (chg[p].before != run) ok = false; }
            run = chg[p].after;
            above = run;
            ++cnt;
            ++p;
        }
        const uint32_t fm = is_int4(h->qmin, h->qmax) ? 0xFu : 0xFFu;
        uint32_t meta = (uint32_t)(below & fm) | ((uint32_t)(above & fm) << 8) | (cnt > 1 ? 0x10000u : 0u);
        const float t = cnt == 0 ? __int_as_float(0x7f800000) : thr;   // +inf: never reached
        cells[i] = make_uint2(__float_as_uint(t), meta);
    }
    if (run != h->code_hi || p != n) ok = false;
    h->valid = ok ? 1 : 0;
}

// compact table from the sorted change list (run after finalize_kernel)
__global__ void finalize4_kernel(Header* h, Header4* h4, uint32_t* cells4, const Change* chg) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Header4 v{};
    const int n = h->nchg;
    bool ok = is_int4(h->qmin, h->qmax) && n <= kMaxChanges;
    if (n >= 2) {
        const float lo = chg[0].y, hi = chg[n - 1].y;
        v.a = __fdiv_rn(1.0f, hi - lo);
        v.b = __fmaf_rn(-lo, v.a, 0.5f / 255.0f);
    } else if (n == 1) {
        v.a = 1.0f;
        v.b = __fadd_rn(0.5f, -chg[0].y);
    }
    if (!(v.a >= 0.0f && v.a < 3.0e38f)) ok = false;
    int run = h->code_lo;
    int p = 0;
    // A cell may hold a cluster of change points (gelu_pinned(y)/s is not
    // monotone at the ulp level, so a code can flicker c, c+1, c, c+1 over a
    // few floats): one word covers it when every point of the cluster lies in
    // one 256-float run R (see above), where the epilogue evaluates
    // directly; below / above R the codes are the cluster's first "before"
    // and last "after" (the verify pass re-checks every float).
    auto in_win = [](uint32_t b, uint32_t wb) { return b - wb < 256u; };
    for (int i = 0; i < kCells4 && ok; ++i) {
        uint32_t w = 0x7F800000u | (uint32_t)(run & 0xF) * 0x11u;
        const int before = run;
        int cnt = 0;
        uint32_t fb = 0, lb = 0;
        while (p < n && (int)cell4(chg[p].y, v.a, v.b) == i) {
            if (chg[p].before != run) ok = false;
            if (cnt == 0) fb = __float_as_uint(chg[p].y);
            lb = __float_as_uint(chg[p].y);
            run = chg[p].after;
            ++cnt;
            ++p;
        }
        if (cnt >= 1) {
            uint32_t wb = fb & ~0xFFu;
            if (!(in_win(fb, wb) && in_win(lb, wb))) wb = lb & ~0xFFu;
            if (!(in_win(fb, wb) && in_win(lb, wb))) ok = false;
            if ((wb & 0x7FFFFFFFu) < 256u) ok = false;   // F - 256 would cross zero (denormal thresholds)
            w = (wb - 256u) | (uint32_t)(before & 0xF) | ((uint32_t)(run & 0xF) << 4);
        }
        cells4[i] = w;
    }
    if (run != h->code_hi || p != n) ok = false;
    v.valid = ok ? 1 : 0;
    *h4 = v;
}

// every float of the scanned ranges: lookup4 decision == direct evaluation
__global__ void verify4_kernel(const Header* h, Header4* h4, const uint32_t* cells4, uint32_t bp0, uint32_t np,
                               uint32_t bn0, uint32_t nn) {
    if (!h4->valid) return;
    const float a = h4->a, b = h4->b;
    const int gelu = h->gelu, qmin = h->qmin, qmax = h->qmax;
    const float s = h->s_out;
    const uint32_t total = np + nn;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        const float y = k < np ? range_y(0, bp0, np, k) : range_y(1, bn0, nn, k - np);
        uint32_t f;
        if (lookup4(cells4[cell4(y, a, b)], y, &f)) continue;
        if (f != ((uint32_t)direct_code(y, gelu, s, qmin, qmax) & 0xFu)) {
            h4->valid = 0;
            return;
        }
    }
}

__global__ void verify_kernel(Header* h, const uint2* cells, uint32_t bp0, uint32_t np, uint32_t bn0, uint32_t nn) {
    if (!h->valid) return;
    const Header hh = *h;
    const uint32_t total = np + nn;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        const float y = k < np ? range_y(0, bp0, np, k) : range_y(1, bn0, nn, k - np);
        if (lookup(hh, cells, y) != direct_code(y, hh.gelu, hh.s_out, hh.qmin, hh.qmax)) {
            h->valid = 0;
            return;
        }
    }
}

}  // namespace rq
}  // namespace mkq
