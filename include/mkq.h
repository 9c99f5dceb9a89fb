/*
 * mkq.h -- C ABI of the B200-native MKQ-BERT W4A4 inference hot path
 *          (arXiv 2203.13483, "MKQ-BERT: Quantized BERT with 4-bits Weights
 *          and Activations").  Library: paper_2203_13483_b200/libmkq.so.
 *
 * Citations: "P:n" = line n of the paper text;
 * "Rn" = a reading of the paper recorded in DESIGN.md §3; "§8a-x" = a row of
 * the hot-path scope table in SURVEY.md §8(a).
 *
 * Conventions shared by every entry point
 * ----------------------------------------
 *  - Pointers marked [device] are CUDA device pointers; pointers marked
 *    [host] are read during the call only.  The caller owns every buffer; the
 *    library never allocates, frees or synchronizes device memory, except a
 *    process-wide cache of TMA descriptors keyed by (pointer, shape, stride)
 *    (descriptors encode no contents, so allocator reuse is safe).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call
 *    only enqueues work on it and returns; the sequence is CUDA-graph
 *    capturable.  Asynchronous faults surface at the caller's next sync.
 *  - Matrices are row-major.  "K-major" operands store the reduction index
 *    contiguously.  int4 codes are packed two per byte: element k of a row is
 *    in byte k/2, even k in the low nibble, two's complement (layout D2, R12).
 *  - Errors: arguments are validated in the order NULL -> SHAPE -> ALIGN ->
 *    SCALE -> RANGE -> DEVICE before anything is enqueued; on error nothing
 *    is launched and the status is returned (detail: mkq_last_error()).  The
 *    only device accepted is compute capability 10.0 (B200, sm_100a); there
 *    is no fallback of any kind.
 *  - Calls are thread-safe; mkq_last_error() is thread-local.
 */
#ifndef MKQ_H
#define MKQ_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MKQ_API __attribute__((visibility("default")))
#else
#define MKQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MKQ_OK = 0,
    MKQ_ERR_NULL = 1,      /* a required pointer is NULL                         */
    MKQ_ERR_SHAPE = 2,     /* dimension out of range / not a multiple required   */
    MKQ_ERR_ALIGN = 3,     /* pointer or leading dimension misaligned            */
    MKQ_ERR_SCALE = 4,     /* scale <= 0 or not finite (S:136 reading, R14)      */
    MKQ_ERR_RANGE = 5,     /* qmin/qmax/bits/mode not representable / unknown    */
    MKQ_ERR_DEVICE = 6,    /* current device is not compute capability 10.0      */
    MKQ_ERR_WORKSPACE = 7, /* workspace too small                                */
    MKQ_ERR_CUDA = 8       /* a CUDA runtime/driver call failed                  */
} mkq_status;

/* Largest reduction length: the tensor-core accumulator holds 256*sum(a*w)
 * for int4 operands (see mkq_gemm_w4a4) and |a*w| <= 2^14 for int8, so
 * K * 2^14 < 2^31 keeps every int32 accumulator exact. */
#define MKQ_MAX_K 131040

MKQ_API const char *mkq_status_string(int status);
MKQ_API const char *mkq_last_error(void);     /* thread-local detail of the last error */
MKQ_API int mkq_version(void);                /* 10000*major + 100*minor + patch        */

/* Epilogue output modes (§8a-a4..a6; R11). */
typedef enum {
    MKQ_OUT_F32 = 0,   /* fp32 y = dequant [+GELU]                               */
    MKQ_OUT_BF16 = 1,  /* bf16, round-to-nearest-even of the fp32 value          */
    MKQ_OUT_I32 = 2,   /* raw exact int32 accumulators sum_k a*w (no dequant)    */
    MKQ_OUT_I4 = 3,    /* requantized int4 codes (packed, D2) with s_out (a6)    */
    MKQ_OUT_I8 = 4,    /* requantized int8 codes with s_out (a6)                 */
    MKQ_OUT_F16 = 5    /* fp16, round-to-nearest-even of the fp32 value          */
} mkq_out;

/* Fused epilogue description [host].  For each output (m, n):
 *   acc  = sum_k a[m,k] * w[n,k]                         (exact int32)
 *   sc   = fl32(s_a * s_w[n])
 *   y    = bias ? fmaf((float)acc, sc, bias[n]) : fl32((float)acc * sc)     (R4)
 *   y    = gelu ? gelu_pinned(y) : y                      (P:98 GELU; R7)
 *   out  = mode F32/BF16/F16: y;  I4/I8: clamp(rint_even(y / s_out), qmin_out,
 *          qmax_out)                                      (Eq.1; R1-R3)
 * A NULL epilogue pointer means {MKQ_OUT_F32, gelu 0}. */
typedef struct {
    int32_t out;       /* mkq_out                                          */
    int32_t gelu;      /* 0 or 1; ignored for MKQ_OUT_I32                  */
    float s_out;       /* requantization scale (I4/I8 only), > 0, finite   */
    int32_t qmin_out;  /* requantization code range (I4/I8 only)           */
    int32_t qmax_out;
    /* Optional [device] table from mkq_requant_table() built for exactly
     * (gelu, s_out, qmin_out, qmax_out); NULL = evaluate gelu_pinned and the
     * division per output.  Results are bit-identical either way (the table
     * is exact by construction and self-verified; an invalid table is
     * ignored on the device). */
    const void *requant_table;
} mkq_epilogue;

/* Bytes of a requant table (device buffer, caller-owned, 16-byte aligned). */
MKQ_API size_t mkq_requant_table_size(void);

/* Build the exact y-space lookup table of the fused requantize epilogue
 * (§8a-a5/a6; DESIGN.md §5 "requant table"):  for every fp32 y,
 *     code(y) = clamp(rint_even((gelu ? gelu_pinned(y) : y) / s_out), qmin, qmax)
 * is tabulated as per-cell thresholds, found by evaluating code(y) for every
 * float where it can change.  Asynchronous on `stream`; needs
 * qmin <= 0 <= qmax.  The table depends only on (gelu, s_out, qmin, qmax). */
MKQ_API mkq_status mkq_requant_table(int gelu, float s_out, int qmin, int qmax, void *table,
                                     size_t table_bytes, void *stream);

/* ------------------------------------------------------------------------
 * §8a-a1: activation (or weight) quantize + pack, Eq.1:
 *   q[r, c] = clamp(rint_even(x[r, c] / s), qmin, qmax),  s = scale[0]
 *   (per_row = 0, per-tensor) or scale[r] (per_row = 1, "per-row").
 * x      [device] fp32 [rows, cols], row stride ldx_elems (>= cols).
 * scale  [device] fp32, 1 value or `rows` values.  Values are NOT inspected
 *        on the host (device memory); they must be > 0 and finite.
 * bits   4 -> q is packed int4 [rows, cols/2] (cols even); 8 -> int8.
 * qmin/qmax: code range; int4 within [-8, 7], int8 within [-128, 127],
 *        qmin < qmax (e.g. activations [-8,7], weights [-7,7]; R1).
 * q      [device] codes, row stride ldq_bytes (>= packed row bytes).
 * rows == 0 or cols == 0 is a valid no-op.
 * ---------------------------------------------------------------------- */
MKQ_API mkq_status mkq_quantize_pack(const float *x, int64_t rows, int64_t cols, int64_t ldx_elems,
                             const float *scale, int per_row, int bits, int qmin, int qmax,
                             void *q, int64_t ldq_bytes, void *stream);

/* §8a-a0: max-abs scale ("maximum of the absolute value", normalised by
 * l_max, R6; floor 1e-8):  s = max(max|x| / l_max, 1e-8) per row (per_row=1,
 * s_out[rows]) or per tensor (per_row=0, s_out[1]).  x [device] fp32. */
MKQ_API mkq_status mkq_absmax_scale(const float *x, int64_t rows, int64_t cols, int64_t ldx_elems,
                            int per_row, float l_max, float *s_out, void *stream);

/* ------------------------------------------------------------------------
 * §8a-a2..a6: W4A4 quantized linear layer  out = epi(A W^T).
 * a   [device] packed int4 activation codes [M, K/2], row stride lda_bytes.
 * w   [device] packed int4 weight codes [N, K/2] (one row per output
 *     channel, K-major), row stride ldw_bytes.
 * s_a per-tensor activation scale (> 0, finite).
 * s_w [device] fp32 [N] per-output-channel weight scales.
 * bias[device] fp32 [N] or NULL.
 * out [device] output [M, N] in the epilogue's mode, row stride ldo_bytes
 *     (I4: packed [M, N/2]).
 * Shape rules: M >= 0 (0 = no-op); N % 32 == 0; K % 32 == 0, 32 <= K <=
 * MKQ_MAX_K.  Alignment: a, w, out 16-byte aligned; lda/ldw/ldo multiples of
 * 16 bytes and >= the packed row size.  Every code of a and w must be a valid
 * int4 (any nibble is); results are exact (the GPU accumulates 256*sum(a*w)
 * in int32 and shifts right by 8).
 * ws/ws_bytes: workspace, may be NULL/0 when mkq_gemm_workspace_size() == 0.
 * ---------------------------------------------------------------------- */
MKQ_API mkq_status mkq_gemm_w4a4(const void *a, int64_t lda_bytes, const void *w, int64_t ldw_bytes,
                         int64_t M, int64_t N, int64_t K, float s_a, const float *s_w,
                         const float *bias, const mkq_epilogue *epi, void *out,
                         int64_t ldo_bytes, void *ws, size_t ws_bytes, void *stream);

/* §8a-a7: W8A8 variant for the paper's mixed 4/8-bit layers:
 * identical contract with int8 codes a [M, K], w [N, K] (K % 32 == 0). */
MKQ_API mkq_status mkq_gemm_w8a8(const void *a, int64_t lda_bytes, const void *w, int64_t ldw_bytes,
                         int64_t M, int64_t N, int64_t K, float s_a, const float *s_w,
                         const float *bias, const mkq_epilogue *epi, void *out,
                         int64_t ldo_bytes, void *ws, size_t ws_bytes, void *stream);

/* Workspace of mkq_gemm_w4a4 / mkq_gemm_w8a8 for an (M, N, K) call: 0 (no
 * workspace is needed).  For small M (the paper's Table
 * 2 regime) the library splits K over the CTAs of a thread-block cluster and
 * sums the exact int32 partials (R15) through distributed shared memory. */
MKQ_API size_t mkq_gemm_workspace_size(int64_t M, int64_t N, int64_t K);

/* NEXT(4) fused glue (the residual + post-LN of P:79-100 / R9
 * fused into the W4A4 GEMM that produces its input):
 *   y = LN(fma((float)acc, fl(s_a*s_w[n]), b[n]) + res; gamma, beta, eps)
 *   [+ q = Eq.1 codes of y with (s_q, q_bits, qmin, qmax)]
 * acc as mkq_gemm_w4a4 (a [M, K] packed int4 codes, w [N, K] packed int4);
 * res, y [device] fp32 [M, N] (row strides ldr / ldy elements, 16-byte
 * aligned rows); gamma, beta [device] fp32 [N]; q [device] packed codes
 * [M, N*q_bits/8] (row stride ldq bytes, 16-byte aligned; q_bits 0 = none).
 * N = 256 * np, np in [1, 4] (hidden 256..1024), K % 32 == 0.  LN statistics
 * are the two-pass mean / centred variance of residual_ln (fp32, different
 * summation order: results agree with mkq_gemm_w4a4 + mkq_residual_layernorm
 * within LN rounding, and are deterministic).  ws >=
 * mkq_gemm_residual_ln_workspace_size(M, N) bytes (row-statistics exchange
 * between the CTAs of a row; the call zeroes its counters on `stream`).
 * Two kernels, same contract: for small M (ceil(M/128) co-resident clusters of
 * N/64 CTAs, e.g. the paper's Table-2 batches) one thread-block cluster per
 * 128-row block exchanges the row statistics over distributed shared memory
 * and does not touch ws; otherwise CTA pairs exchange them through ws. */
MKQ_API size_t mkq_gemm_residual_ln_workspace_size(int64_t M, int64_t N);
MKQ_API mkq_status mkq_gemm_residual_ln(const void *a, int64_t lda_bytes, const void *w, int64_t ldw_bytes,
                                        int64_t M, int64_t N, int64_t K, float s_a, const float *s_w,
                                        const float *bias, const float *res, int64_t ldr, const float *gamma,
                                        const float *beta, float eps, float *y, int64_t ldy, int q_bits,
                                        float s_q, int qmin, int qmax, void *q, int64_t ldq, void *ws,
                                        size_t ws_bytes, void *stream);

/* NEXT(4) fused communication for the column-parallel FFN:
 * the FFN1 GEMM of one rank (W4A4, GELU + int4 requantize through the compact
 * table, epi->out = MKQ_OUT_I4 with epi->requant_table) stores every output
 * tile directly into the gathered FFN2-input buffer of every rank at column
 * col0 (this rank's block), instead of a local output + NCCL all-gather:
 *   outs[g]     [device, valid in this process: the local buffer or a peer's
 *               CUDA-IPC mapping] packed int4 [M, >= col0 + N], row stride
 *               ldo bytes (16-byte multiple);
 *   counters[g] [device, same] uint32: after all its stores are complete each
 *               CTA adds 1 to every counters[g] (release, system scope); a
 *               launch adds mkq_gemm_gather_arrivals(M, N) per counter.
 * N % 256 == 0, K <= 1024 (the FFN1 shape).  The consumer blocks its stream
 * with mkq_wait_counter(own counter, target) before reading its buffer.
 * Reusing a gathered buffer needs the peers' readers to be done with it
 * (the caller's barrier).  Codes are bit-identical to mkq_gemm_w4a4. */
MKQ_API int mkq_gemm_gather_arrivals(int64_t M, int64_t N);
MKQ_API mkq_status mkq_gemm_w4a4_gather(const void *a, int64_t lda_bytes, const void *w, int64_t ldw_bytes,
                                        int64_t M, int64_t N, int64_t K, float s_a, const float *s_w,
                                        const float *bias, const mkq_epilogue *epi, void *const *outs, int nout,
                                        int64_t col0, int64_t ldo_bytes, uint32_t *const *counters, void *stream);
/* Block `stream` until *counter >= target (acquire, system scope). */
MKQ_API mkq_status mkq_wait_counter(const uint32_t *counter, uint32_t target, void *stream);
/* CUDA IPC plumbing for the peer buffers.  get_handle writes the 64-byte
 * handle of the allocation containing dev_ptr and dev_ptr's byte offset in
 * it; a peer maps the allocation with open_handle (-> *base; the buffer is
 * base + offset) and unmaps it with close(base).  Errors: MKQ_ERR_NULL,
 * MKQ_ERR_CUDA (message in mkq_last_error()). */
MKQ_API mkq_status mkq_ipc_get_handle(const void *dev_ptr, void *handle64, int64_t *offset);
MKQ_API mkq_status mkq_ipc_open_handle(const void *handle64, void **base);
MKQ_API mkq_status mkq_ipc_close(void *base);

/* Diagnostics / tests: GEMM tile plan for small M.  -1 = heuristic (default;
 * also the MKQ_SMALL_M environment variable), 0 = never the small-M plan,
 * 1 = always the tcgen05 cluster split-K plan, 2 = always the mma.sync
 * small-M kernel.  Results are identical in every mode. */
MKQ_API void mkq_set_small_m_mode(int mode);

/* ------------------------------------------------------------------------
 * §8a-a8 glue (★s): multi-head self-attention core, Eq.3-5 (with
 * the q.v^T typo read as q.k^T, R8):  OA = softmax(q k^T / sqrt(d_k)) v,
 * per sequence and head; softmax in fp32.
 * qkv  [device] fp16 [tokens, 3*heads*head_dim] = [q | k | v], head a at
 *      columns a*head_dim of each block; row stride ld_qkv_elems.
 * cu_seqlens [device] int32 [batch+1] prefix sums of sequence lengths
 *      (packed "valid tokens", R13) or NULL = `batch` sequences of
 *      `seq` tokens.  max_seq bounds every length (<= 1024).
 * out_mode MKQ_OUT_F32 (fp32 OA [tokens, heads*head_dim]) or MKQ_OUT_I4 /
 *      MKQ_OUT_I8 (OA quantized with s_out, fused; packed like mkq_quantize_pack).
 * head_dim must be 64.
 * ---------------------------------------------------------------------- */
MKQ_API mkq_status mkq_attention(const void *qkv, int64_t ld_qkv_elems, int64_t batch, int64_t max_seq,
                         const int32_t *cu_seqlens, int64_t tokens, int heads, int head_dim,
                         int out_mode, float s_out, int qmin, int qmax, void *out,
                         int64_t ldo_bytes, void *stream);

/* integer attention core for short sequences (reading
 * R19; Eq.3-5).  qkv [device] int8 codes [tokens, 3*heads*64] =
 * [q | k | v] (Eq.1 of the QKV GEMM output with the per-tensor scale s_qkv,
 * codes in [-127, 127]; the MKQ_OUT_I8 epilogue of mkq_gemm_*), row stride
 * ld_qkv_bytes.  Per sequence and head:
 *   S_ij = q_i . k_j (exact int32);  c = fl32(fl32(s_qkv*s_qkv) / 8);
 *   p_ij = rint_even(255 * exp(-c * (max_j S_ij - S_ij)))  (fp64 exp, uint8);
 *   OA_i = fl32(fl32(fl32(sum_j p_ij v_j) / fl32(sum_j p_ij)) * s_qkv).
 * Every step but the fp64 exp is exact; results equal the oracle bit for bit
 * unless 255*exp(.) falls within an ulp of a half-integer.  max_seq <= 128,
 * head_dim 64; cu_seqlens / out_mode / s_out / qmin / qmax as mkq_attention. */
MKQ_API mkq_status mkq_attention_i8(const void *qkv, int64_t ld_qkv_bytes, int64_t batch, int64_t max_seq,
                                    const int32_t *cu_seqlens, int64_t tokens, int heads, int head_dim,
                                    float s_qkv, int out_mode, float s_out, int qmin, int qmax, void *out,
                                    int64_t ldo_bytes, void *stream);

/* §8a-a8 glue: y = LayerNorm(x + res) * g + b (post-LN, eps, fp32; R9), and
 * optionally (bits = 4 or 8, else 0) the fused Eq.1 quantize of y with the
 * per-tensor scale s_q into q (packed like mkq_quantize_pack).
 * x, res, y [device] fp32 [rows, cols] (row strides ld_elems); res may be
 * NULL; g, b [device] fp32 [cols]; cols % 4 == 0, cols <= 8192. */
MKQ_API mkq_status mkq_residual_layernorm(const float *x, const float *res, int64_t rows, int64_t cols,
                                  int64_t ld_elems, const float *g, const float *b, float eps,
                                  float *y, int bits, float s_q, int qmin, int qmax, void *q,
                                  int64_t ldq_bytes, void *stream);

/* Column-parallel FFN plumbing: an NCCL all_gather of per-rank
 * column blocks yields src = [g][rows][cb] bytes (rank-major); this writes
 * dst[row][r*cb + j] = src[r][row][j] with row stride ld_dst bytes.
 * src/dst [device], 16-byte aligned, cb % 16 == 0, ld_dst >= g*cb. */
MKQ_API mkq_status mkq_interleave_blocks(const void *src, void *dst, int64_t g, int64_t rows, int64_t cb,
                                         int64_t ld_dst_bytes, void *stream);

/* ------------------------------------------------------------------------
 * QAT-side fake quantization with the §4.1 scale
 * gradients, one HBM pass over a contiguous fp32 tensor x [n]:
 *   q_i   = clamp(rint_even(x_i / s), qmin, qmax)       Eq.1, R1-R3
 *   y_i   = fl32(s * q_i)                                fake-quant Q[x]
 *   clip_i: rint_even(x_i / s) lies outside [qmin, qmax]  (R18)
 *   grad_x_i = clip_i ? 0 : grad_y_i                     STE input gradient (R18)
 *   grad_s[0] = sum_i (clip_i ? q_i : q_i - x_i / s)     STE scale gradient (
 *                                                         LSQ rule for clipped x_i, R17)
 *   grad_s[1] = 2 sum_i (s q_i - x_i) q_i                MSE scale gradient
 * scale  [device] fp32, 1 value (> 0, finite; not inspected on the host).
 * y, grad_x [device] fp32 [n] or NULL (not computed); grad_y [device] fp32 [n],
 *        required with grad_x.  grad_s [device] fp64 [2] or NULL.
 * ws     [device] >= mkq_fake_quant_workspace_size(n) bytes, 16-byte aligned
 *        (per-block partial sums; the final fold is in a fixed order, so
 *        grad_s is deterministic).  The fp64 sums equal the oracle's up to
 *        summation order; y and grad_x are bit-exact.
 * qmin < qmax within [-128, 127] (any bit width <= 8).  n == 0: grad_s = 0.
 * ---------------------------------------------------------------------- */
MKQ_API size_t mkq_fake_quant_workspace_size(int64_t n);
MKQ_API mkq_status mkq_fake_quant(const float *x, int64_t n, const float *scale, int qmin, int qmax,
                                  float *y, const float *grad_y, float *grad_x, double *grad_s,
                                  void *ws, size_t ws_bytes, void *stream);

/* activation-scale calibration on the GPU, P:72 ("top
 * 0.01% largest value ... as the initial scale", normalised by l_max, R6):
 *   a = |x| sorted ascending; pos = p (n-1); lo = floor(pos);
 *   hi = min(lo+1, n-1); quant = fl32(a[lo] + (pos-lo)(a[hi]-a[lo])) (fp64);
 *   *s_out = fl32(quant / l_max).
 * The order statistics are exact (radix select on the bit patterns of |x|,
 * no sort, no host copy); bit-identical to the definition.
 * x [device] fp32 [n], n >= 1, finite.  p in [0, 1] (0.9999 in the paper).
 * s_out [device] fp32 [1].  ws [device] >= mkq_act_scale_workspace_size()
 * bytes, 16-byte aligned. */
MKQ_API size_t mkq_act_scale_workspace_size(void);
MKQ_API mkq_status mkq_act_scale(const float *x, int64_t n, double p, float l_max, float *s_out,
                                 void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * One quantized post-LN BERT encoder layer (§8a rows a1-a8 composed):
 *   c   = Q(h; s_qkv_in)                                   a1
 *   qkv = f16( Linear_{W^{QKV}}(c) )                        a2-a4
 *         (int_attention: Q(Linear(c); s_attn), int8 codes)
 *   OA  = Attention(qkv) -> Q(.; s_o_in)                    a8 (fused quantize;
 *         int_attention: mkq_attention_i8)
 *   o   = Linear_{W^A}(.) (+b^A), fp32                      a2-a4
 *   h1  = LN1(o + h) -> fp32 and Q(h1; s_ffn1_in)           a8 + a1 fused
 *   a2  = Q(GELU(Linear_{W^1}(.)); s_ffn2_in)               a2-a6 (fused)
 *   f   = Linear_{W^2}(a2), fp32                            a2-a4
 *   out = LN2(f + h1)                                        a8
 * bits = 4 (W4A4: every GEMM mkq_gemm_w4a4, codes [-8,7], weights packed
 * int4) or 8 (W8A8: mkq_gemm_w8a8, codes [-128,127], weights int8).
 * Weights [device] are [N, K] K-major: W^{QKV} [3h, h], W^A [h, h],
 * W^1 [ffn, h], W^2 [h, ffn]; row stride = K*bits/8 bytes.
 * hidden % 64 == 0 (heads*64 == hidden), ffn % 32 == 0.
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t hidden, heads, ffn, bits;
    const void *w_qkv, *w_o, *w_1, *w_2;
    const float *sw_qkv, *sw_o, *sw_1, *sw_2;
    const float *b_qkv, *b_o, *b_1, *b_2;
    const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
    float s_qkv_in, s_o_in, s_ffn1_in, s_ffn2_in;
    float ln_eps;
    /* optional [device] mkq_requant_table(1, s_ffn2_in, qmin, qmax) for the
     * FFN1 epilogue (NULL = direct evaluation; identical results) */
    const void *ffn1_requant_table;
    /* NEXT(2): 1 = integer attention core (R19): the QKV epilogue emits int8
     * codes [-127, 127] with the per-tensor scale s_attn and attention runs
     * mkq_attention_i8 (max_seq <= 128); 0 = fp16 q|k|v (R10). */
    int32_t int_attention;
    float s_attn;
    /* NEXT(4) fused glue across a layer stack (optional; NULL / 0 = off):
     * in_codes  [device] the Eq.1 codes of h_in with (s_qkv_in, bits), packed as
     *           mkq_quantize_pack writes them ([tokens, hidden*bits/8], row
     *           stride hidden*bits/8 bytes, 16-byte aligned): the input
     *           quantize (a1) is skipped -- the previous layer's LN2 wrote them;
     * out_codes [device] LN2 also writes the Eq.1 codes of h_out with
     *           (s_out_codes, out_bits in {4, 8}; codes [-8,7] / [-128,127])
     *           in that layout: the next layer's in_codes.  Bit-identical to
     *           quantizing h_out separately (the LN kernel's fused quantize).
     * in_codes may equal out_codes (the QKV GEMM reads it before LN2 writes). */
    const void *in_codes;
    void *out_codes;
    float s_out_codes;
    int32_t out_bits;
} mkq_layer;

/* 1 if mkq_bert_layer runs the W^A + LN1 and W^2 + LN2 stages as
 * mkq_gemm_residual_ln (W4A4, hidden in {256, 512, 768, 1024}, tokens >=
 * 4096), 0 if as mkq_gemm_w4a4/w8a8 + mkq_residual_layernorm. */
MKQ_API int mkq_layer_fused_ln(const mkq_layer *L, int64_t tokens);

/* Workspace bytes for `tokens` rows (intermediates of one layer). */
MKQ_API size_t mkq_bert_layer_workspace_size(const mkq_layer *L, int64_t tokens);

/* h_in, h_out [device] fp32 [tokens, hidden] (may alias: in-place is
 * allowed).  cu_seqlens as for mkq_attention (NULL = batch x seq; then
 * tokens must equal batch*seq). */
MKQ_API mkq_status mkq_bert_layer(const mkq_layer *L, const float *h_in, int64_t batch, int64_t max_seq,
                          const int32_t *cu_seqlens, int64_t tokens, float *h_out, void *ws,
                          size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MKQ_H */
