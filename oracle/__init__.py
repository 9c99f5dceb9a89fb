"""CPU oracle for the MKQ-BERT W4A4 BERT-layer hot path (arXiv 2203.13483).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares
no code with the CUDA path (paper_2203_13483_b200/) and never imports it.

Two parts:
  * ``mkq_oracle.c`` -- scalar C for every bit-exact step (Eq.1 quantizer,
    int4 packing, int32 GEMM, dequant, gelu_pinned, requant, bf16/f16
    rounding, weight calibration, the §4.1 scale gradients);
  * ``layer.py``     -- the fp64 NumPy BERT layer glue (attention, residual
    + LayerNorm) that composes the C steps into one post-LN layer.

Every function cites the PAPER.md line (P:n) or DESIGN.md reading (Rn) it
follows.  "Parity unpinned" items are listed in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mkq_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared",
          "-fPIC", "-Wall"]


def build(force: bool = False) -> str:
    """Compile mkq_oracle.c -> liboracle.so (gcc, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        F = ctypes.c_float
        L.oracle_quantize.argtypes = [P, I64, I64, I64, P, I, I, I, P]
        L.oracle_fake_quant.argtypes = [P, I64, F, I, I, P]
        L.oracle_pack_int4.argtypes = [P, I64, I64, P, I64]
        L.oracle_unpack_int4.argtypes = [P, I64, I64, I64, P]
        L.oracle_gemm_i32.argtypes = [P, P, I64, I64, I64, P]
        L.oracle_dequant.argtypes = [P, I64, I64, F, P, P, P]
        L.oracle_erf_pinned.argtypes = [F]
        L.oracle_erf_pinned.restype = F
        L.oracle_gelu_pinned.argtypes = [F]
        L.oracle_gelu_pinned.restype = F
        L.oracle_gelu_array.argtypes = [P, I64, P]
        L.oracle_f32_to_bf16.argtypes = [F]
        L.oracle_f32_to_bf16.restype = ctypes.c_uint16
        L.oracle_f32_to_f16.argtypes = [F]
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_linear.argtypes = [P, P, I64, I64, I64, F, P, P, I, I, F, I, I, P]
        L.oracle_absmax_scale.argtypes = [P, I64, I64, I64, I, F, P]
        L.oracle_scale_grad_ste.argtypes = [P, I64, F, I, I]
        L.oracle_scale_grad_ste.restype = ctypes.c_double
        L.oracle_scale_grad_mse.argtypes = [P, I64, F, I, I]
        L.oracle_scale_grad_mse.restype = ctypes.c_double
        L.oracle_ste_grad_x.argtypes = [P, P, I64, F, I, I, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _chk(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


# Output modes of oracle_linear (mirrors the product's epilogue list, R11).
OUT_F32, OUT_BF16, OUT_I32, OUT_I4, OUT_I8, OUT_F16 = 0, 1, 2, 3, 4, 5

# Code ranges (reading R1).
A4 = (-8, 7)      # int4 activations, BJ.north_star clip(x/s, -8, 7)
W4 = (-7, 7)      # int4 weights, max-abs calibration maps to +-7
A8 = (-128, 127)  # int8 activations
W8 = (-127, 127)  # int8 weights


def quantize(x, scale, qmin, qmax, per_row=False) -> np.ndarray:
    """Eq.1: codes = round(clamp(x/s)), fp32 division, ties-even."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    assert x.ndim == 2
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(scale, dtype=np.float32)))
    if per_row:
        assert s.shape[0] == x.shape[0]
    q = np.empty(x.shape, dtype=np.int8)
    _chk(lib().oracle_quantize(_p(x), x.shape[0], x.shape[1], x.shape[1], _p(s),
                               int(per_row), qmin, qmax, _p(q)), "quantize")
    return q


def fake_quant(x, s, qmin, qmax) -> np.ndarray:
    """Q[x] = s * round(clamp(x/s)) (Eq.1)."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    out = np.empty_like(x)
    _chk(lib().oracle_fake_quant(_p(x), x.size, float(np.float32(s)), qmin, qmax, _p(out)),
         "fake_quant")
    return out


def pack_int4(q) -> np.ndarray:
    """Layout D2 / reading R12: byte k/2 of a row, even k in the low nibble."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    rows, cols = q.shape
    out = np.zeros((rows, cols // 2), dtype=np.uint8)
    _chk(lib().oracle_pack_int4(_p(q), rows, cols, _p(out), cols // 2), "pack_int4")
    return out


def unpack_int4(p, cols) -> np.ndarray:
    p = np.ascontiguousarray(p, dtype=np.uint8)
    rows = p.shape[0]
    q = np.empty((rows, cols), dtype=np.int8)
    _chk(lib().oracle_unpack_int4(_p(p), rows, cols, p.shape[1], _p(q)), "unpack_int4")
    return q


def gemm_i32(qa, qw) -> np.ndarray:
    """acc = qa @ qw^T summed exactly."""
    qa = np.ascontiguousarray(qa, dtype=np.int8)
    qw = np.ascontiguousarray(qw, dtype=np.int8)
    M, K = qa.shape
    N = qw.shape[0]
    assert qw.shape[1] == K
    acc = np.empty((M, N), dtype=np.int32)
    _chk(lib().oracle_gemm_i32(_p(qa), _p(qw), M, N, K, _p(acc)), "gemm_i32")
    return acc


def dequant(acc, s_a, s_w, bias=None) -> np.ndarray:
    """y = fma((float)acc, fl(s_a*s_w[n]), b[n]) (reading R4)."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    M, N = acc.shape
    s_w = np.ascontiguousarray(s_w, dtype=np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    y = np.empty((M, N), dtype=np.float32)
    _chk(lib().oracle_dequant(_p(acc), M, N, float(np.float32(s_a)), _p(s_w),
                              None if b is None else _p(b), _p(y)), "dequant")
    return y


def gelu_pinned(y) -> np.ndarray:
    """Reading R7: fp32 exact-erf GELU with the frozen erf polynomial."""
    y = np.ascontiguousarray(y, dtype=np.float32)
    g = np.empty_like(y)
    lib().oracle_gelu_array(_p(y), y.size, _p(g))
    return g


def erf_pinned(t: float) -> float:
    return lib().oracle_erf_pinned(float(t))


def f32_to_bf16_bits(x) -> np.ndarray:
    f = lib().oracle_f32_to_bf16
    x = np.asarray(x, dtype=np.float32)
    return np.array([f(float(v)) for v in x.ravel()], dtype=np.uint16).reshape(x.shape)


def f32_to_f16_bits(x) -> np.ndarray:
    f = lib().oracle_f32_to_f16
    x = np.asarray(x, dtype=np.float32)
    return np.array([f(float(v)) for v in x.ravel()], dtype=np.uint16).reshape(x.shape)


def linear(qa, qw, s_a, s_w, bias=None, mode=OUT_F32, gelu=False, s_out=1.0,
           qmin_out=-8, qmax_out=7) -> np.ndarray:
    """One quantized linear layer from its definition: a3 -> a4 -> [a5] -> out.

    Modes: OUT_F32 fp32; OUT_BF16 / OUT_F16 uint16 bit patterns (RN-even of the
    fp32 value); OUT_I32 raw accumulators; OUT_I4 / OUT_I8 requantized codes
    (unpacked int8, a6 with s_out)."""
    qa = np.ascontiguousarray(qa, dtype=np.int8)
    qw = np.ascontiguousarray(qw, dtype=np.int8)
    M, K = qa.shape
    N = qw.shape[0]
    s_w = np.ascontiguousarray(s_w, dtype=np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    dt = {OUT_F32: np.float32, OUT_BF16: np.uint16, OUT_F16: np.uint16,
          OUT_I32: np.int32, OUT_I4: np.int8, OUT_I8: np.int8}[mode]
    out = np.empty((M, N), dtype=dt)
    _chk(lib().oracle_linear(_p(qa), _p(qw), M, N, K, float(np.float32(s_a)), _p(s_w),
                             None if b is None else _p(b), mode, int(gelu),
                             float(np.float32(s_out)), qmin_out, qmax_out, _p(out)),
         "linear")
    return out


def absmax_scale(w, l_max, per_row=True) -> np.ndarray:
    """P:72 max-abs calibration normalised by l_max (R6), floor 1e-8."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    rows, cols = w.shape
    s = np.empty(rows if per_row else 1, dtype=np.float32)
    lib().oracle_absmax_scale(_p(w), rows, cols, cols, int(per_row), float(l_max), _p(s))
    return s


def scale_grad_ste(x, s, qmin=-8, qmax=7) -> float:
    """§4.1.1: sum_i(-x_i/s + round(x_i/s)); clipped elements
    contribute their clamped code (LSQ, reading R17)."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    return lib().oracle_scale_grad_ste(_p(x), x.size, float(np.float32(s)), qmin, qmax)


def scale_grad_mse(x, s, qmin=-8, qmax=7) -> float:
    """§4.1.2: 2 sum_i (Q[x_i]-x_i) round(x_i/s)."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    return lib().oracle_scale_grad_mse(_p(x), x.size, float(np.float32(s)), qmin, qmax)


def ste_grad_x(x, grad_y, s, qmin=-8, qmax=7) -> np.ndarray:
    """STE input gradient: grad_y where x is not clipped, else 0 (R18)."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    gy = np.ascontiguousarray(grad_y, dtype=np.float32).ravel()
    assert gy.size == x.size
    out = np.empty_like(x)
    _chk(lib().oracle_ste_grad_x(_p(x), _p(gy), x.size, float(np.float32(s)), qmin, qmax, _p(out)),
         "ste_grad_x")
    return out


def abs_quantile(x, p=0.9999) -> np.float32:
    """Calibration statistic (P:72 'top 0.01% largest value'): the p-quantile
    of |x| by sorting, linear interpolation between order statistics
    (reading R6/O-S), rounded once to fp32."""
    a = np.sort(np.abs(np.asarray(x, dtype=np.float64)).ravel())
    pos = p * (a.size - 1)
    lo = int(np.floor(pos))
    hi = min(lo + 1, a.size - 1)
    frac = pos - lo
    return np.float32(a[lo] + frac * (a[hi] - a[lo]))


def act_scale(x, l_max=7, p=0.9999) -> np.float32:
    """s_a = quantile_p(|x|) / l_max (R6), fp32 division."""
    return np.float32(abs_quantile(x, p)) / np.float32(l_max)
