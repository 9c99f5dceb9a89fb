/*
 * mkq_oracle.c -- plain, slow, obviously-correct CPU oracle for the MKQ-BERT
 * W4A4 / W8A8 linear-layer hot path (arXiv 2203.13483).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * under paper_2203_13483_b200/; constants that the specification fixes (the
 * gelu_pinned coefficients of DESIGN.md R7) are typed here independently.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (x86-64 SSE arithmetic; no x87, no FMA contraction, IEEE defaults).
 *
 * Citations are to /root/reference/PAPER.md lines ("P:n", with the section /
 * equation) and to DESIGN.md readings ("R1".."R16").
 *
 * Pins (tests/test_oracle.py): every function below is pinned by something
 * other than itself -- the paper's worked example, hand-worked
 * tables (tests/golden/), closed forms, invariants and brute force.  The only
 * function pinned by tolerance alone is gelu_pinned (against fp64 erf).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <fenv.h>

#define OK 0
#define ERR_RANGE 4
#define ERR_OVERFLOW 9

/* --------------------------------------------------------------------- */
/* Eq.1 quantizer (§3.1): q = round(clamp(x/s, l_min, l_max)).    */
/* Reading R1: int4 activations l in [-8,7], weights [-7,7] (qmin/qmax are */
/* passed explicitly).  R2: ties to even (nearbyintf under FE_TONEAREST).  */
/* R3: x/s is one IEEE binary32 division.  Rounding is monotone and fixes  */
/* integers, so clamp-after-round equals Eq.1's round(clamp(.)).           */
/* --------------------------------------------------------------------- */
static int8_t quant1(float x, float s, int qmin, int qmax)
{
    float v = x / s;            /* binary32 division, round-to-nearest */
    float r = nearbyintf(v);    /* ties to even under FE_TONEAREST */
    if (r < (float)qmin) r = (float)qmin;
    if (r > (float)qmax) r = (float)qmax;
    return (int8_t)(int)r;
}

/* Quantize a [rows, cols] fp32 matrix (row stride ldx elements) with one
 * per-tensor scale (per_row = 0) or one scale per row (per_row = 1, P:68
 * "per-row scale").  Codes are written unpacked, one int8 per element,
 * row-major [rows, cols]. */
int oracle_quantize(const float *x, int64_t rows, int64_t cols, int64_t ldx,
                    const float *scale, int per_row, int qmin, int qmax,
                    int8_t *q)
{
    if (fegetround() != FE_TONEAREST) return ERR_RANGE;
    for (int64_t i = 0; i < rows; ++i) {
        float s = per_row ? scale[i] : scale[0];
        for (int64_t j = 0; j < cols; ++j)
            q[i * cols + j] = quant1(x[i * ldx + j], s, qmin, qmax);
    }
    return OK;
}

/* Fake-quant value Q[x] = s * q (Eq.1), one fp32 multiply. */
int oracle_fake_quant(const float *x, int64_t n, float s, int qmin, int qmax,
                      float *out)
{
    for (int64_t i = 0; i < n; ++i)
        out[i] = s * (float)quant1(x[i], s, qmin, qmax);
    return OK;
}

/* --------------------------------------------------------------------- */
/* int4 packing (reading R12, layout D2): element k of a row lives in byte */
/* k/2; even k in the low nibble; two's-complement nibbles.               */
/* --------------------------------------------------------------------- */
int oracle_pack_int4(const int8_t *q, int64_t rows, int64_t cols, uint8_t *out,
                     int64_t ld_bytes)
{
    if (cols % 2) return ERR_RANGE;
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t k = 0; k < cols; k += 2) {
            int lo = q[i * cols + k], hi = q[i * cols + k + 1];
            if (lo < -8 || lo > 7 || hi < -8 || hi > 7) return ERR_RANGE;
            out[i * ld_bytes + k / 2] = (uint8_t)((lo & 0xF) | ((hi & 0xF) << 4));
        }
    return OK;
}

int oracle_unpack_int4(const uint8_t *p, int64_t rows, int64_t cols,
                       int64_t ld_bytes, int8_t *q)
{
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t k = 0; k < cols; ++k) {
            uint8_t b = p[i * ld_bytes + k / 2];
            int nib = (k % 2 == 0) ? (b & 0xF) : (b >> 4);
            q[i * cols + k] = (int8_t)(nib >= 8 ? nib - 16 : nib);
        }
    return OK;
}

/* --------------------------------------------------------------------- */
/* Integer GEMM ("int4 matrix multiplication"):               */
/*   acc[m][n] = sum_k qa[m][k] * qw[n][k]                                 */
/* summed in int64 and checked to fit int32 (the GPU accumulates in s32). */
/* --------------------------------------------------------------------- */
int oracle_gemm_i32(const int8_t *qa, const int8_t *qw, int64_t M, int64_t N,
                    int64_t K, int32_t *acc)
{
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int64_t k = 0; k < K; ++k)
                s += (int64_t)qa[m * K + k] * (int64_t)qw[n * K + k];
            if (s > INT32_MAX || s < INT32_MIN) return ERR_OVERFLOW;
            acc[m * N + n] = (int32_t)s;
        }
    return OK;
}

/* --------------------------------------------------------------------- */
/* Dequant (reading R4): real value s_a*s_w[n]*acc + b[n] (P:66 s*q, */
/* P:98 bias).  fp32 op order: sc = fl(s_a*s_w[n]); y = fma((float)acc,   */
/* sc, b[n]); without bias y = fl((float)acc * sc).                       */
/* --------------------------------------------------------------------- */
static float dequant1(int32_t acc, float s_a, float s_wn, const float *bias,
                      int64_t n)
{
    float sc = s_a * s_wn;
    float a = (float)acc;  /* RN conversion */
    return bias ? fmaf(a, sc, bias[n]) : a * sc;
}

int oracle_dequant(const int32_t *acc, int64_t M, int64_t N, float s_a,
                   const float *s_w, const float *bias, float *y)
{
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n)
            y[m * N + n] = dequant1(acc[m * N + n], s_a, s_w[n], bias, n);
    return OK;
}

/* --------------------------------------------------------------------- */
/* gelu_pinned (reading R7): the FFN activation of P:98, "GELU" computed  */
/* in float32, fixed as the exact-erf GELU 0.5*y*(1+erf(y/sqrt2)) */
/* with erf replaced by the frozen piecewise polynomial of DESIGN.md R7   */
/* (coefficients typed here from DESIGN.md, hex-exact binary32).          */
/* --------------------------------------------------------------------- */
static const float GP[7] = {   /* P, degree 6 .. 0, in u = t*t, t < 1 */
    0x1.4fd528p-14f, -0x1.a63f9ep-11f, 0x1.545360p-8f, -0x1.b80286p-6f,
    0x1.ce2d7cp-4f, -0x1.812740p-2f, 0x1.20dd76p+0f};
static const float GQ[13] = {  /* Q, degree 12 .. 0, in u = t - 2.5, 1 <= t < 3.92 */
    0x1.3db5fep-17f, -0x1.5d0ec2p-16f, -0x1.0bd2eep-14f, 0x1.23355ep-12f,
    -0x1.280846p-12f, -0x1.29eb5ap-11f, 0x1.70d992p-9f, -0x1.901754p-8f,
    0x1.1a5d5cp-7f, -0x1.11b3b0p-7f, 0x1.64ef0ap-8f, -0x1.1d7db8p-9f,
    0x1.aab4b4p-12f};

float oracle_erf_pinned(float t)   /* t >= 0 */
{
    if (t < 1.0f) {
        float u = t * t;
        float p = GP[0];
        for (int i = 1; i < 7; ++i) p = fmaf(p, u, GP[i]);
        return t * p;
    }
    if (t < 3.92f) {
        float u = t - 2.5f;
        float q = GQ[0];
        for (int i = 1; i < 13; ++i) q = fmaf(q, u, GQ[i]);
        return 1.0f - q;
    }
    return 1.0f;
}

float oracle_gelu_pinned(float y)
{
    float t = fabsf(y) * 0x1.6a09e6p-1f;   /* fl32(1/sqrt(2)) */
    float e = oracle_erf_pinned(t);
    if (y < 0.0f) e = -e;
    float h = 0.5f * y;                     /* exact */
    return fmaf(h, e, h);                   /* h*(1+e), one rounding */
}

int oracle_gelu_array(const float *y, int64_t n, float *g)
{
    for (int64_t i = 0; i < n; ++i) g[i] = oracle_gelu_pinned(y[i]);
    return OK;
}

/* --------------------------------------------------------------------- */
/* bf16 / f16 conversion of an fp32 value, round-to-nearest-even (R11).    */
/* --------------------------------------------------------------------- */
uint16_t oracle_f32_to_bf16(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

/* fp32 -> IEEE binary16, round-to-nearest-even, with subnormals and      */
/* overflow to infinity: written from the binary16 definition.           */
uint16_t oracle_f32_to_f16(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
    uint32_t a = u & 0x7fffffffu;
    if (a > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);   /* NaN */
    if (a == 0x7f800000u) return (uint16_t)(sign | 0x7c00u);  /* inf */
    double v = (double)f;                  /* exact */
    if (v < 0) v = -v;
    /* binary16: value = m * 2^(e-24) for the representable grid; find the */
    /* spacing (ulp) of the binade containing v, round v/ulp to even.      */
    int e;
    frexp(v, &e);                          /* v = f * 2^e, 0.5 <= f < 1 */
    int exp16 = e - 1;                     /* v in [2^exp16, 2^(exp16+1)) */
    if (exp16 < -14) exp16 = -14;          /* subnormal spacing 2^-24 */
    double ulp = ldexp(1.0, exp16 - 10);
    double n = nearbyint(v / ulp);         /* exact division by a power of two */
    double r = n * ulp;
    if (r >= 65520.0 || r > 65504.0) return (uint16_t)(sign | 0x7c00u);
    /* encode r */
    if (r == 0.0) return sign;
    int er;
    frexp(r, &er);
    int E = er - 1;
    if (E < -14) {                         /* subnormal */
        return (uint16_t)(sign | (uint16_t)(r / ldexp(1.0, -24)));
    }
    uint32_t mant = (uint32_t)(r / ldexp(1.0, E - 10)) - 1024u;
    return (uint16_t)(sign | (uint16_t)((E + 15) << 10) | (uint16_t)mant);
}

/* --------------------------------------------------------------------- */
/* The whole linear layer of one GEMM, spelled out from its definition:   */
/*   codes (unpacked int8) -> acc (a3) -> y (a4) -> [gelu (a5)] ->        */
/*   output mode: 0 f32, 1 bf16, 2 raw i32, 3 int4 codes, 4 int8 codes    */
/*   (a6 requant with s_out, qmin_out, qmax_out), 5 f16 (see below).      */
/* Output for modes 3/4 is written unpacked (int8 per element).          */
/* --------------------------------------------------------------------- */
int oracle_linear(const int8_t *qa, const int8_t *qw, int64_t M, int64_t N,
                  int64_t K, float s_a, const float *s_w, const float *bias,
                  int mode, int gelu, float s_out, int qmin_out, int qmax_out,
                  void *out)
{
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int64_t k = 0; k < K; ++k)
                s += (int64_t)qa[m * K + k] * (int64_t)qw[n * K + k];
            if (s > INT32_MAX || s < INT32_MIN) return ERR_OVERFLOW;
            int32_t acc = (int32_t)s;
            if (mode == 2) { ((int32_t *)out)[m * N + n] = acc; continue; }
            float y = dequant1(acc, s_a, s_w[n], bias, n);
            if (gelu) y = oracle_gelu_pinned(y);
            switch (mode) {
            case 0: ((float *)out)[m * N + n] = y; break;
            case 1: ((uint16_t *)out)[m * N + n] = oracle_f32_to_bf16(y); break;
            case 5: ((uint16_t *)out)[m * N + n] = oracle_f32_to_f16(y); break;
            case 3:
            case 4: ((int8_t *)out)[m * N + n] = quant1(y, s_out, qmin_out, qmax_out); break;
            default: return ERR_RANGE;
            }
        }
    return OK;
}

/* Weight calibration ("maximum of the absolute value for each weight  */
/* tensor", reading R6: normalised by l_max; per output row, R5), floor    */
/* 1e-8 for an all-zero row: s = max(max_k |w[n,k]| / l_max, 1e-8).        */
int oracle_absmax_scale(const float *w, int64_t rows, int64_t cols, int64_t ld,
                        int per_row, float l_max, float *s)
{
    float gmax = 0.0f;
    for (int64_t i = 0; i < rows; ++i) {
        float mx = 0.0f;
        for (int64_t j = 0; j < cols; ++j) {
            float a = fabsf(w[i * ld + j]);
            if (a > mx) mx = a;
        }
        if (per_row) {
            float v = mx / l_max;
            s[i] = v < 1e-8f ? 1e-8f : v;
        }
        if (mx > gmax) gmax = mx;
    }
    if (!per_row) {
        float v = gmax / l_max;
        s[0] = v < 1e-8f ? 1e-8f : v;
    }
    return OK;
}

/* QAT-side gradients of §4.1 (NEXT(3) in SURVEY §8f).                     */
/* "Clipped" = the unclamped code rint(x/s) lies outside [qmin, qmax]      */
/* (reading R18).                                                          */
static int clipped1(float x, float s, int qmin, int qmax)
{
    float r = nearbyintf(x / s);
    return r < (float)qmin || r > (float)qmax;
}

/* STE scale gradient: sum_i (-x_i/s + round(x_i/s)), the     */
/* derivation of "previous work" [kdlsq, esser2019learned].  The   */
/* paper's derivation ignores the clamp; for a clipped x_i, Q[x_i] =       */
/* s*qmax (or s*qmin), whose derivative is the clamped code itself (LSQ's  */
/* rule) -- reading R17.  Summed in double.                                */
double oracle_scale_grad_ste(const float *x, int64_t n, float s, int qmin, int qmax)
{
    double g = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        int q = quant1(x[i], s, qmin, qmax);
        if (clipped1(x[i], s, qmin, qmax))
            g += (double)q;
        else
            g += -(double)x[i] / (double)s + (double)q;
    }
    return g;
}

/* MSE scale gradient: 2 * sum_i (Q[x_i] - x_i) * round(x_i/s) */
/* with round(.) the clamped code (Eq.1): Q_{s+ds}[x] = (s+ds) q holds for */
/* clipped elements too.  Summed in double.                                */
double oracle_scale_grad_mse(const float *x, int64_t n, float s, int qmin, int qmax)
{
    double g = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        int q = quant1(x[i], s, qmin, qmax);
        double Q = (double)s * (double)q;
        g += (Q - (double)x[i]) * (double)q;
    }
    return 2.0 * g;
}

/* STE input gradient ("d round / d . = 1"): dL/dx_i = dL/dQ_i where */
/* x_i is not clipped, 0 where it is (reading R18; LSQ / PyTorch           */
/* fake-quant convention -- the paper is silent on the clamp).             */
int oracle_ste_grad_x(const float *x, const float *grad_y, int64_t n, float s,
                      int qmin, int qmax, float *grad_x)
{
    for (int64_t i = 0; i < n; ++i)
        grad_x[i] = clipped1(x[i], s, qmin, qmax) ? 0.0f : grad_y[i];
    return OK;
}
