"""fp64 NumPy oracle of one post-LN BERT layer with quantized linears.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Composition (§3.2; readings R8-R10 of DESIGN.md):
  qkv  = Linear_{W^{Q,K,V}}(Q(h))                         P:87   (Eq.3)
  A    = softmax(q k^T / sqrt(d_k))                        P:88   (Eq.4, R8: q k^T)
  OA   = A v ; heads concatenated                          P:89-93 (Eq.5)
  o    = Linear_{W^A}(Q(OA)) + b^A
  h1   = LN(o + h)                (post-LN, eps 1e-12)      R9
  f    = Linear_{W^2}(Q(GELU(Linear_{W^1}(Q(h1)))))
  out  = LN(f + h1)                                        R9
where Q is Eq.1 with the static per-tensor activation scale, every
Linear is the integer GEMM + dequant of oracle.linear, GELU is gelu_pinned
(R7) fused with the requantize of the FFN2 input (a5, a6), LayerNorm and
softmax are computed in float64 (P:234 asks for >= float32) and attention
takes q, k, v as the fp32 dequant outputs of the QKV linear (SURVEY §8(c)
O-L; P:234 keeps the glue in float32).  The product's fp16 attention
operands (R10) are a product property with their own stated
tolerance in the GPU tests; they are not mirrored here.

Parity status: the bit-exact linear steps are pinned in tests/test_oracle.py;
the fp64 glue (attention, LN) is pinned by closed forms (softmax rows sum to
1, uniform attention on equal keys, LN mean 0 / variance 1) and by a
brute-force per-element loop on tiny inputs.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (A4, A8, W4, W8, OUT_F32, OUT_I4, OUT_I8, absmax_scale,
               act_scale, linear, quantize)

LN_EPS = 1e-12


def act_range(bits: int):
    return A4 if bits == 4 else A8


def weight_range(bits: int):
    return W4 if bits == 4 else W8


@dataclass
class QWeight:
    """a0 weight prep (R5/R6): per-output-row max-abs scale."""
    codes: np.ndarray      # int8 [N, K] (unpacked codes)
    s_w: np.ndarray        # fp32 [N]
    bias: np.ndarray       # fp32 [N]


def prepare_weight(w: np.ndarray, bias: np.ndarray, bits: int) -> QWeight:
    lo, hi = weight_range(bits)
    s_w = absmax_scale(w, hi, per_row=True)
    codes = quantize(w, s_w, lo, hi, per_row=True)
    return QWeight(codes, s_w, np.asarray(bias, dtype=np.float32))


@dataclass
class LayerWeights:
    hidden: int
    heads: int
    ffn: int
    bits: int
    qkv: QWeight
    o: QWeight
    w1: QWeight
    w2: QWeight
    ln1_g: np.ndarray
    ln1_b: np.ndarray
    ln2_g: np.ndarray
    ln2_b: np.ndarray
    # static activation scales (learned by QAT in the paper; calibrated here)
    s_qkv_in: np.float32 = np.float32(1)
    s_o_in: np.float32 = np.float32(1)
    s_ffn1_in: np.float32 = np.float32(1)
    s_ffn2_in: np.float32 = np.float32(1)
    # NEXT(2) integer attention core (R19): scale of the int8 q|k|v codes;
    # None = float attention on the fp32 q|k|v (SURVEY O-L)
    s_attn: object = None


def layernorm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = LN_EPS) -> np.ndarray:
    """Row LayerNorm in float64: (x - mean) / sqrt(var + eps) * g + b."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * np.asarray(g, np.float64) + np.asarray(b, np.float64)


def softmax(s: np.ndarray) -> np.ndarray:
    """Row softmax in float64, max-subtracted."""
    s = np.asarray(s, dtype=np.float64)
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def attention_int8(codes: np.ndarray, seqlens, heads: int, s_qkv) -> np.ndarray:
    """NEXT(2) integer attention core (reading R19 of DESIGN.md),
    Eq.3-5 on int8 codes of q | k | v with one per-tensor scale
    s_qkv (Eq.1 of the QKV output, codes in [-127, 127]):
        S_ij  = q_i . k_j                       exact integers
        c     = fl32(fl32(s_qkv * s_qkv) * 1/8)  (1/sqrt(d_k), d_k = 64, exact)
        d_ij  = max_j' S_ij' - S_ij              integers >= 0
        p_ij  = rint_even(255 * exp(-c d_ij))    fp64, uint8; p = 255 at the row max
        OA_i  = fl32(fl32(fl32(sum_j p_ij v_j) / fl32(sum_j p_ij)) * s_qkv)
    softmax(c S) v with the probabilities held as 8-bit integers; every step
    but the fp64 exp is exact integer arithmetic, and the final ratio is one
    fp32 division (|sum p v| <= 255*127*128 < 2^24 for L <= 128).
    codes: int8 [M, 3d]; returns OA fp32 [M, d]."""
    codes = np.asarray(codes, dtype=np.int64)
    M, three_d = codes.shape
    d = three_d // 3
    dk = d // heads
    assert dk == 64
    s = np.float32(s_qkv)
    c = np.float32(np.float32(s * s) * np.float32(0.125))
    out = np.zeros((M, d), dtype=np.float32)
    r0 = 0
    for L in seqlens:
        rows = slice(r0, r0 + L)
        for a in range(heads):
            cols = slice(a * dk, (a + 1) * dk)
            q = codes[rows, 0 * d:1 * d][:, cols]
            k = codes[rows, 1 * d:2 * d][:, cols]
            v = codes[rows, 2 * d:3 * d][:, cols]
            S = q @ k.T                                          # exact int64
            dd = S.max(axis=1, keepdims=True) - S                # >= 0
            p = np.rint(255.0 * np.exp(-(np.float64(c) * dd.astype(np.float64)))).astype(np.int64)
            num = p @ v                                          # exact
            den = p.sum(axis=1, keepdims=True)
            y = (num.astype(np.float32) / den.astype(np.float32)).astype(np.float32)
            out[rows, cols] = (y * s).astype(np.float32)
        r0 += L
    assert r0 == M
    return out


def attention(qkv: np.ndarray, seqlens, heads: int) -> np.ndarray:
    """Eq.3-5 per sequence and head, fp64.

    qkv: [M, 3d] with columns [q | k | v], head a at columns a*d_k:(a+1)*d_k
    of each block.  seqlens: lengths of the consecutive sequences packed in
    the M rows (padding removed, reading R13).  Returns OA [M, d] (float64)."""
    qkv = np.asarray(qkv, dtype=np.float64)
    M, three_d = qkv.shape
    d = three_d // 3
    dk = d // heads
    out = np.zeros((M, d), dtype=np.float64)
    r0 = 0
    for L in seqlens:
        rows = slice(r0, r0 + L)
        for a in range(heads):
            c = slice(a * dk, (a + 1) * dk)
            q = qkv[rows, 0 * d:1 * d][:, c]
            k = qkv[rows, 1 * d:2 * d][:, c]
            v = qkv[rows, 2 * d:3 * d][:, c]
            A = softmax(q @ k.T / np.sqrt(dk))
            out[rows, c] = A @ v
        r0 += L
    assert r0 == M
    return out


@dataclass
class LayerTrace:
    codes_in: np.ndarray = None
    qkv: np.ndarray = None        # fp32 q|k|v (int8 codes with s_attn)
    oa: np.ndarray = None         # fp32
    codes_oa: np.ndarray = None
    o: np.ndarray = None          # fp32 (W^A output incl. bias)
    h1: np.ndarray = None         # fp32
    codes_h1: np.ndarray = None
    codes_ffn2_in: np.ndarray = None
    f: np.ndarray = None          # fp32
    h_out: np.ndarray = None      # fp32
    extra: dict = field(default_factory=dict)


def bert_layer(h: np.ndarray, W: LayerWeights, seqlens) -> LayerTrace:
    """One quantized post-LN BERT layer; returns every intermediate."""
    T = LayerTrace()
    lo, hi = act_range(W.bits)
    h = np.asarray(h, dtype=np.float32)
    T.codes_in = quantize(h, W.s_qkv_in, lo, hi)
    if W.s_attn is not None:   # NEXT(2): Eq.1 of the QKV output to int8, integer attention (R19)
        T.qkv = linear(T.codes_in, W.qkv.codes, W.s_qkv_in, W.qkv.s_w, W.qkv.bias, mode=OUT_I8,
                       s_out=W.s_attn, qmin_out=-127, qmax_out=127)
        T.oa = attention_int8(T.qkv, seqlens, W.heads, W.s_attn)
    else:
        T.qkv = linear(T.codes_in, W.qkv.codes, W.s_qkv_in, W.qkv.s_w, W.qkv.bias, mode=OUT_F32)
        T.oa = attention(T.qkv.astype(np.float64), seqlens, W.heads).astype(np.float32)
    T.codes_oa = quantize(T.oa, W.s_o_in, lo, hi)
    T.o = linear(T.codes_oa, W.o.codes, W.s_o_in, W.o.s_w, W.o.bias, mode=OUT_F32)
    T.h1 = layernorm(T.o.astype(np.float64) + h, W.ln1_g, W.ln1_b).astype(np.float32)
    T.codes_h1 = quantize(T.h1, W.s_ffn1_in, lo, hi)
    T.codes_ffn2_in = linear(T.codes_h1, W.w1.codes, W.s_ffn1_in, W.w1.s_w, W.w1.bias,
                             mode=OUT_I4 if W.bits == 4 else OUT_I8, gelu=True,
                             s_out=W.s_ffn2_in, qmin_out=lo, qmax_out=hi)
    T.f = linear(T.codes_ffn2_in, W.w2.codes, W.s_ffn2_in, W.w2.s_w, W.w2.bias, mode=OUT_F32)
    T.h_out = layernorm(T.f.astype(np.float64) + T.h1, W.ln2_g, W.ln2_b).astype(np.float32)
    return T


def calibrate(h_calib: np.ndarray, W: LayerWeights, seqlens, int_attention: bool = False) -> LayerWeights:
    """Sequential calibration of the static activation scales
    (P:72 'top 0.01% largest value', P:121 calibration step; R6/O-S):
    each scale is set from the layer's own activations on a calibration
    batch, in pipeline order, using the scales already fixed upstream
    (int_attention: also s_attn = p99.99(|q|k|v|) / 127, R19)."""
    lo, hi = act_range(W.bits)
    h = np.asarray(h_calib, dtype=np.float32)
    W.s_qkv_in = act_scale(h, hi)
    codes = quantize(h, W.s_qkv_in, lo, hi)
    if int_attention:
        qkv32 = linear(codes, W.qkv.codes, W.s_qkv_in, W.qkv.s_w, W.qkv.bias, mode=OUT_F32)
        W.s_attn = act_scale(qkv32, 127)
        qkv8 = linear(codes, W.qkv.codes, W.s_qkv_in, W.qkv.s_w, W.qkv.bias, mode=OUT_I8, s_out=W.s_attn,
                      qmin_out=-127, qmax_out=127)
        oa = attention_int8(qkv8, seqlens, W.heads, W.s_attn)
    else:
        qkv = linear(codes, W.qkv.codes, W.s_qkv_in, W.qkv.s_w, W.qkv.bias, mode=OUT_F32)
        oa = attention(qkv.astype(np.float64), seqlens, W.heads).astype(np.float32)
    W.s_o_in = act_scale(oa, hi)
    o = linear(quantize(oa, W.s_o_in, lo, hi), W.o.codes, W.s_o_in, W.o.s_w, W.o.bias)
    h1 = layernorm(o.astype(np.float64) + h, W.ln1_g, W.ln1_b).astype(np.float32)
    W.s_ffn1_in = act_scale(h1, hi)
    g = linear(quantize(h1, W.s_ffn1_in, lo, hi), W.w1.codes, W.s_ffn1_in, W.w1.s_w,
               W.w1.bias, mode=OUT_F32, gelu=True)
    W.s_ffn2_in = act_scale(g, hi)
    return W
