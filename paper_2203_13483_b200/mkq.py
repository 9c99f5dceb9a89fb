"""Thin PyTorch binding over the C ABI (include/mkq.h): argument marshalling
only.  Every function is named after the C entry point it calls; every step
of the hot path runs in libmkq.so's CUDA kernels.  Tensors must live on a
CUDA device (a B200); nothing here computes on the host.
"""
from __future__ import annotations

import ctypes
from collections import OrderedDict
from typing import Optional, Tuple

import torch

from ._lib import (OUT_BF16, OUT_F16, OUT_F32, OUT_I32, OUT_I4, OUT_I8, MkqEpilogue, MkqLayer,
                   check, lib)

__all__ = ["mkq_requant_table", "mkq_quantize_pack", "mkq_absmax_scale", "mkq_gemm_w4a4", "mkq_gemm_w8a8",
           "mkq_attention", "mkq_residual_layernorm", "mkq_bert_layer", "mkq_gemm_residual_ln", "mkq_interleave_blocks", "mkq_fake_quant",
           "mkq_act_scale", "mkq_attention_i8", "out_dtype_bytes",
           "OUT_F32", "OUT_BF16", "OUT_I32", "OUT_I4", "OUT_I8", "OUT_F16"]


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("mkq: tensors must be CUDA tensors (no host fallback)")
    return ctypes.c_void_p(t.data_ptr())


def _row_bytes(t: torch.Tensor) -> int:
    assert t.dim() == 2 and t.stride(1) == 1, "row-major 2-D tensor with unit column stride required"
    return t.stride(0) * t.element_size()


def out_dtype_bytes(mode: int):
    return {OUT_F32: (torch.float32, 4), OUT_I32: (torch.int32, 4), OUT_BF16: (torch.bfloat16, 2),
            OUT_F16: (torch.float16, 2), OUT_I8: (torch.int8, 1), OUT_I4: (torch.uint8, 0.5)}[mode]


def mkq_quantize_pack(x: torch.Tensor, scale: torch.Tensor, bits: int = 4, qmin: int = -8, qmax: int = 7,
                      per_row: bool = False, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Eq.1 quantize + pack (§8a-a1).  x fp32 [rows, cols]; scale fp32 device
    tensor with 1 (per-tensor) or rows (per-row) values."""
    rows, cols = x.shape
    if out is None:
        out = torch.empty((rows, cols // 2 if bits == 4 else cols),
                          dtype=torch.uint8 if bits == 4 else torch.int8, device=x.device)
    check("mkq_quantize_pack", lib().mkq_quantize_pack(
        _ptr(x), rows, cols, x.stride(0), _ptr(scale), int(per_row), bits, qmin, qmax, _ptr(out),
        _row_bytes(out), _stream(stream)))
    return out


def mkq_absmax_scale(x: torch.Tensor, l_max: float, per_row: bool = True, out: Optional[torch.Tensor] = None,
                     stream=None) -> torch.Tensor:
    """a0 calibration: s = max(max|x| / l_max, 1e-8) per row or per tensor."""
    rows, cols = x.shape
    if out is None:
        out = torch.empty(rows if per_row else 1, dtype=torch.float32, device=x.device)
    check("mkq_absmax_scale", lib().mkq_absmax_scale(_ptr(x), rows, cols, x.stride(0), int(per_row),
                                                     float(l_max), _ptr(out), _stream(stream)))
    return out


def mkq_fake_quant(x: torch.Tensor, scale: torch.Tensor, qmin: int = -8, qmax: int = 7, grad_y=None,
                   want_y: bool = True, want_grad_s: bool = True, ws: Optional[torch.Tensor] = None, stream=None):
    """§4.1 QAT step: fake-quant y = s*q, STE input gradient
    (given grad_y) and the STE / MSE scale gradients, one HBM pass.
    Returns (y | None, grad_x | None, grad_s fp64 [2] = {STE, MSE} | None)."""
    assert x.is_contiguous() and x.dtype == torch.float32
    n = x.numel()
    y = torch.empty_like(x) if want_y else None
    gx = torch.empty_like(x) if grad_y is not None else None
    if grad_y is not None:
        assert grad_y.is_contiguous() and grad_y.shape == x.shape
    gs = torch.empty(2, dtype=torch.float64, device=x.device) if want_grad_s else None
    nb = int(lib().mkq_fake_quant_workspace_size(n))
    if ws is None or ws.numel() < nb:
        ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
    check("mkq_fake_quant", lib().mkq_fake_quant(_ptr(x), n, _ptr(scale), qmin, qmax, _ptr(y), _ptr(grad_y),
                                                 _ptr(gx), _ptr(gs), _ptr(ws), ws.numel(), _stream(stream)))
    return y, gx, gs


def mkq_act_scale(x: torch.Tensor, l_max: float = 7.0, p: float = 0.9999, out: Optional[torch.Tensor] = None,
                  ws: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """P:72 calibration on the GPU: fl32(quantile_p(|x|)) / l_max (R6), an
    exact radix select (fp32 device tensor [1])."""
    assert x.is_contiguous() and x.dtype == torch.float32
    if out is None:
        out = torch.empty(1, dtype=torch.float32, device=x.device)
    nb = int(lib().mkq_act_scale_workspace_size())
    if ws is None or ws.numel() < nb:
        ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
    check("mkq_act_scale", lib().mkq_act_scale(_ptr(x), x.numel(), float(p), float(l_max), _ptr(out), _ptr(ws),
                                               ws.numel(), _stream(stream)))
    return out


_TABLES: "OrderedDict" = OrderedDict()
_TABLES_MAX = 64   # LRU bound: QAT / calibration loops build one table per distinct s_out


def mkq_requant_table(gelu: bool, s_out: float, qmin: int, qmax: int, device=None, stream=None,
                      cache: bool = True) -> torch.Tensor:
    """Exact y-space lookup table of the fused (GELU +) requantize epilogue,
    built on the device by libmkq (mkq_requant_table).  The build stream is
    synchronized once before the table is returned, so a cached table is
    complete for consumers on any stream."""
    device = torch.device(device if device is not None else "cuda")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    key = (bool(gelu), float(s_out), int(qmin), int(qmax), str(device))
    if cache and key in _TABLES:
        _TABLES.move_to_end(key)
        return _TABLES[key]
    nbytes = int(lib().mkq_requant_table_size())
    t = torch.empty(nbytes, dtype=torch.uint8, device=device)
    st = stream if stream is not None else torch.cuda.current_stream(device)
    check("mkq_requant_table", lib().mkq_requant_table(int(gelu), float(s_out), qmin, qmax, _ptr(t), nbytes,
                                                       _stream(st)))
    st.synchronize()   # one-off: later readers on other streams see a complete table
    if cache:
        _TABLES[key] = t
        while len(_TABLES) > _TABLES_MAX:
            _TABLES.popitem(last=False)
    return t


_GEMM_WS = {}


def _gemm_ws(M: int, N: int, K: int, device, stream):
    """Split-K scratch for small-M GEMMs (mkq_gemm_workspace_size), one
    cached buffer per (device, stream): calls on one stream are ordered."""
    nb = int(lib().mkq_gemm_workspace_size(M, N, K))
    if nb == 0:
        return None
    key = (str(device), _stream(stream).value)
    buf = _GEMM_WS.get(key)
    if buf is None or buf.numel() < nb:
        buf = torch.empty(nb, dtype=torch.uint8, device=device)
        _GEMM_WS[key] = buf
    return buf


def _gemm(name: str, a, w, K: int, s_a: float, s_w, bias, mode: int, gelu: bool, s_out: float, qmin: int,
          qmax: int, out, stream, requant_table=None):
    M, N = a.shape[0], w.shape[0]
    if out is None:
        dt, nb = out_dtype_bytes(mode)
        out = torch.empty((M, int(N * nb) if mode == OUT_I4 else N), dtype=dt, device=a.device)
    if isinstance(requant_table, bool):
        requant_table = mkq_requant_table(gelu, s_out, qmin, qmax, a.device, stream) \
            if (requant_table and mode in (OUT_I4, OUT_I8)) else None
    epi = MkqEpilogue(mode, int(gelu), float(s_out), qmin, qmax,
                      None if requant_table is None else requant_table.data_ptr())
    fn = getattr(lib(), name)
    ws = _gemm_ws(M, N, K, a.device, stream)
    check(name, fn(_ptr(a), _row_bytes(a), _ptr(w), _row_bytes(w), M, N, K, float(s_a), _ptr(s_w), _ptr(bias),
                   ctypes.byref(epi), _ptr(out), _row_bytes(out), _ptr(ws), 0 if ws is None else ws.numel(),
                   _stream(stream)))
    return out


def mkq_gemm_w4a4(a: torch.Tensor, w: torch.Tensor, s_a: float, s_w: torch.Tensor,
                  bias: Optional[torch.Tensor] = None, mode: int = OUT_F32, gelu: bool = False,
                  s_out: float = 1.0, qmin: int = -8, qmax: int = 7, out: Optional[torch.Tensor] = None,
                  K: Optional[int] = None, stream=None, requant_table=True) -> torch.Tensor:
    """W4A4 linear (§8a-a2..a6): a packed [M, K/2], w packed [N, K/2].
    requant_table: True = build/cache the exact requant table (I4/I8 modes),
    False/None = direct evaluation, or a prebuilt table tensor."""
    K = K if K is not None else a.shape[1] * 2
    return _gemm("mkq_gemm_w4a4", a, w, K, s_a, s_w, bias, mode, gelu, s_out, qmin, qmax, out, stream,
                 requant_table)


def mkq_gemm_w8a8(a: torch.Tensor, w: torch.Tensor, s_a: float, s_w: torch.Tensor,
                  bias: Optional[torch.Tensor] = None, mode: int = OUT_F32, gelu: bool = False,
                  s_out: float = 1.0, qmin: int = -128, qmax: int = 127, out: Optional[torch.Tensor] = None,
                  K: Optional[int] = None, stream=None, requant_table=True) -> torch.Tensor:
    """W8A8 linear (§8a-a7): a int8 [M, K], w int8 [N, K]."""
    K = K if K is not None else a.shape[1]
    return _gemm("mkq_gemm_w8a8", a, w, K, s_a, s_w, bias, mode, gelu, s_out, qmin, qmax, out, stream,
                 requant_table)


def mkq_gemm_gather_arrivals(M: int, N: int) -> int:
    """Counter increments one mkq_gemm_w4a4_gather launch adds per buffer."""
    return int(lib().mkq_gemm_gather_arrivals(M, N))


def mkq_gemm_w4a4_gather(a: torch.Tensor, w: torch.Tensor, s_a: float, s_w: torch.Tensor,
                         bias: Optional[torch.Tensor], outs, counters, col0: int, ldo: int, s_out: float,
                         gelu: bool = True, qmin: int = -8, qmax: int = 7, K: Optional[int] = None,
                         requant_table=None, stream=None) -> None:
    """NEXT(4) fused all-gather: the int4-requant W4A4 linear whose tiles land
    in every rank's gathered buffer (mkq_gemm_w4a4_gather).  outs / counters
    are device addresses (ints) valid in this process: local tensors'
    data_ptr() or CUDA-IPC mappings of the peers' buffers."""
    M, N = a.shape[0], w.shape[0]
    K = K if K is not None else a.shape[1] * 2
    if requant_table is None:
        requant_table = mkq_requant_table(gelu, s_out, qmin, qmax, a.device, stream)
    epi = MkqEpilogue(OUT_I4, int(gelu), float(s_out), qmin, qmax, requant_table.data_ptr())
    n = len(outs)
    if len(counters) != n:
        raise ValueError("one counter per gathered buffer")
    outs_c = (ctypes.c_void_p * n)(*[int(o) for o in outs])
    cnt_c = (ctypes.c_void_p * n)(*[int(c) for c in counters])
    check("mkq_gemm_w4a4_gather", lib().mkq_gemm_w4a4_gather(
        _ptr(a), _row_bytes(a), _ptr(w), _row_bytes(w), M, N, K, float(s_a), _ptr(s_w), _ptr(bias),
        ctypes.byref(epi), outs_c, n, int(col0), int(ldo), cnt_c, _stream(stream)))


def mkq_wait_counter(counter: int, target: int, stream=None) -> None:
    """Block `stream` until the uint32 at device address `counter` >= target."""
    check("mkq_wait_counter", lib().mkq_wait_counter(ctypes.c_void_p(int(counter)), target & 0xFFFFFFFF,
                                                     _stream(stream)))


def mkq_ipc_get_handle(t: torch.Tensor) -> Tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, t's byte offset in it)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    check("mkq_ipc_get_handle", lib().mkq_ipc_get_handle(_ptr(t), buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


def mkq_ipc_open_handle(handle: bytes) -> int:
    """Map a peer's allocation; returns its base device address in this process."""
    ptr = ctypes.c_void_p()
    check("mkq_ipc_open_handle", lib().mkq_ipc_open_handle(ctypes.create_string_buffer(bytes(handle), 64),
                                                           ctypes.byref(ptr)))
    return int(ptr.value)


def mkq_ipc_close(base: int) -> None:
    check("mkq_ipc_close", lib().mkq_ipc_close(ctypes.c_void_p(int(base))))


_LN_WS = {}


def mkq_gemm_residual_ln(a: torch.Tensor, w: torch.Tensor, s_a: float, s_w: torch.Tensor,
                         bias: Optional[torch.Tensor], res: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor,
                         eps: float = 1e-12, K: Optional[int] = None, q_bits: int = 0, s_q: float = 1.0,
                         qmin: int = -8, qmax: int = 7, y: Optional[torch.Tensor] = None,
                         q: Optional[torch.Tensor] = None, stream=None):
    """NEXT(4) fused glue: y = LN(W4A4 linear(a) + res) [+ Eq.1 codes of y]
    (mkq_gemm_residual_ln; N = w rows = 256..1024 in steps of 256)."""
    M, N = a.shape[0], w.shape[0]
    K = K if K is not None else a.shape[1] * 2
    if y is None:
        y = torch.empty((M, N), dtype=torch.float32, device=a.device)
    if q_bits and q is None:
        q = torch.empty((M, N // 2 if q_bits == 4 else N), dtype=torch.uint8 if q_bits == 4 else torch.int8,
                        device=a.device)
    nb = int(lib().mkq_gemm_residual_ln_workspace_size(M, N))
    key = (str(a.device), _stream(stream).value)
    ws = _LN_WS.get(key)
    if ws is None or ws.numel() < nb:
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=a.device)
        _LN_WS[key] = ws
    check("mkq_gemm_residual_ln", lib().mkq_gemm_residual_ln(
        _ptr(a), _row_bytes(a), _ptr(w), _row_bytes(w), M, N, K, float(s_a), _ptr(s_w), _ptr(bias), _ptr(res),
        res.stride(0), _ptr(gamma), _ptr(beta), float(eps), _ptr(y), y.stride(0), int(q_bits), float(s_q),
        qmin, qmax, _ptr(q), 0 if q is None else _row_bytes(q), _ptr(ws), ws.numel(), _stream(stream)))
    return (y, q) if q_bits else y


def mkq_attention(qkv: torch.Tensor, heads: int, batch: int, max_seq: int,
                  cu_seqlens: Optional[torch.Tensor] = None, mode: int = OUT_F32, s_out: float = 1.0,
                  qmin: int = -8, qmax: int = 7, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Attention core (Eq.3-5) on fp16 qkv [tokens, 3*hidden]."""
    T = qkv.shape[0]
    hidden = heads * 64
    if out is None:
        if mode == OUT_F32:
            out = torch.empty((T, hidden), dtype=torch.float32, device=qkv.device)
        elif mode == OUT_I4:
            out = torch.empty((T, hidden // 2), dtype=torch.uint8, device=qkv.device)
        else:
            out = torch.empty((T, hidden), dtype=torch.int8, device=qkv.device)
    check("mkq_attention", lib().mkq_attention(
        _ptr(qkv), qkv.stride(0), batch, max_seq, _ptr(cu_seqlens), T, heads, 64, mode, float(s_out), qmin, qmax,
        _ptr(out), _row_bytes(out), _stream(stream)))
    return out


def mkq_attention_i8(qkv: torch.Tensor, heads: int, batch: int, max_seq: int, s_qkv: float,
                     cu_seqlens: Optional[torch.Tensor] = None, mode: int = OUT_F32, s_out: float = 1.0,
                     qmin: int = -8, qmax: int = 7, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """NEXT(2) integer attention core (R19) on int8 qkv codes [tokens, 3*hidden]."""
    T = qkv.shape[0]
    hidden = heads * 64
    if out is None:
        dt, nb = out_dtype_bytes(mode)
        out = torch.empty((T, int(hidden * nb) if mode == OUT_I4 else hidden), dtype=dt, device=qkv.device)
    check("mkq_attention_i8", lib().mkq_attention_i8(
        _ptr(qkv), _row_bytes(qkv), batch, max_seq, _ptr(cu_seqlens), T, heads, 64, float(s_qkv), mode,
        float(s_out), qmin, qmax, _ptr(out), _row_bytes(out), _stream(stream)))
    return out


def mkq_residual_layernorm(x: torch.Tensor, res: Optional[torch.Tensor], g: torch.Tensor, b: torch.Tensor,
                           eps: float = 1e-12, bits: int = 0, s_q: float = 1.0, qmin: int = -8, qmax: int = 7,
                           y: Optional[torch.Tensor] = None, q: Optional[torch.Tensor] = None, stream=None):
    """y = LN(x + res) (post-LN, R9) [+ fused Eq.1 quantize of y].  The C
    call takes one leading dimension for x, res and y, so all three must
    share x's row stride (and have unit column stride)."""
    rows, cols = x.shape
    if y is None:
        y = torch.empty_strided(x.shape, x.stride(), dtype=x.dtype, device=x.device)
    for name, t in (("x", x), ("res", res), ("y", y)):
        if t is not None and (t.shape != x.shape or t.stride(1) != 1 or t.stride(0) != x.stride(0)):
            raise ValueError(f"mkq_residual_layernorm: {name} must be [{rows}, {cols}] with x's row stride "
                             f"{x.stride(0)} and unit column stride")
    if bits and q is None:
        q = torch.empty((rows, cols // 2 if bits == 4 else cols), dtype=torch.uint8 if bits == 4 else torch.int8,
                        device=x.device)
    check("mkq_residual_layernorm", lib().mkq_residual_layernorm(
        _ptr(x), _ptr(res), rows, cols, x.stride(0), _ptr(g), _ptr(b), float(eps), _ptr(y), bits, float(s_q), qmin,
        qmax, _ptr(q), _row_bytes(q) if q is not None else 0, _stream(stream)))
    return (y, q) if bits else y


def mkq_interleave_blocks(src: torch.Tensor, g: int, rows: int, cb: int, out: Optional[torch.Tensor] = None,
                          stream=None) -> torch.Tensor:
    """[g][rows][cb] bytes (rank-major all-gather) -> [rows][g*cb] bytes."""
    if out is None:
        out = torch.empty((rows, g * cb), dtype=torch.uint8, device=src.device)
    check("mkq_interleave_blocks", lib().mkq_interleave_blocks(_ptr(src), _ptr(out), g, rows, cb,
                                                               out.stride(0) * out.element_size(), _stream(stream)))
    return out


class QLayer:
    """Device-resident parameters of one quantized BERT layer (mkq_layer)."""

    FIELDS = ("w_qkv", "w_o", "w_1", "w_2", "sw_qkv", "sw_o", "sw_1", "sw_2", "b_qkv", "b_o", "b_1", "b_2",
              "ln1_g", "ln1_b", "ln2_g", "ln2_b")

    def __init__(self, hidden: int, heads: int, ffn: int, bits: int, tensors: dict, scales: dict,
                 ln_eps: float = 1e-12, use_table: bool = True):
        """scales: s_qkv_in, s_o_in, s_ffn1_in, s_ffn2_in, and optionally s_attn
        (present and > 0 = NEXT(2) integer attention core)."""
        self.hidden, self.heads, self.ffn, self.bits = hidden, heads, ffn, bits
        self.t = {k: tensors[k].contiguous() for k in self.FIELDS}
        self.scales = {k: float(scales[k]) for k in ("s_qkv_in", "s_o_in", "s_ffn1_in", "s_ffn2_in")}
        if scales.get("s_attn"):
            self.scales["s_attn"] = float(scales["s_attn"])
        self.int_attention = "s_attn" in self.scales
        self.ln_eps = ln_eps
        lo, hi = (-8, 7) if bits == 4 else (-128, 127)
        dev = self.t["w_qkv"].device
        self.table = mkq_requant_table(True, self.scales["s_ffn2_in"], lo, hi, dev) if use_table else None
        self.c = MkqLayer(hidden, heads, ffn, bits, *[self.t[k].data_ptr() for k in self.FIELDS],
                          self.scales["s_qkv_in"], self.scales["s_o_in"], self.scales["s_ffn1_in"],
                          self.scales["s_ffn2_in"], float(ln_eps),
                          None if self.table is None else self.table.data_ptr(),
                          int(self.int_attention), float(self.scales.get("s_attn", 0.0)))

    def workspace_size(self, tokens: int) -> int:
        return int(lib().mkq_bert_layer_workspace_size(ctypes.byref(self.c), tokens))

    def fused_ln(self, tokens: int) -> bool:
        """mkq_bert_layer runs W^A + LN1 and W^2 + LN2 as mkq_gemm_residual_ln."""
        return bool(lib().mkq_layer_fused_ln(ctypes.byref(self.c), tokens))


def mkq_bert_layer(layer: QLayer, h_in: torch.Tensor, batch: int, max_seq: int,
                   cu_seqlens: Optional[torch.Tensor] = None, h_out: Optional[torch.Tensor] = None,
                   ws: Optional[torch.Tensor] = None, stream=None, in_codes: Optional[torch.Tensor] = None,
                   out_codes: Optional[torch.Tensor] = None, s_out_codes: float = 0.0,
                   out_bits: int = 0) -> torch.Tensor:
    """One quantized post-LN BERT layer on h_in fp32 [tokens, hidden].
    in_codes: h_in's Eq.1 codes (s_qkv_in, layer.bits), written by the previous
    layer's LN2 (skips the input quantize); out_codes: LN2 also writes h_out's
    codes with (s_out_codes, out_bits) for the next layer (mkq_layer fields)."""
    T = h_in.shape[0]
    if h_out is None:
        h_out = torch.empty_like(h_in)
    need = layer.workspace_size(T)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=h_in.device)
    c = layer.c
    if in_codes is not None or out_codes is not None:
        c = MkqLayer.from_buffer_copy(layer.c)
        c.in_codes = _ptr(in_codes)
        c.out_codes = _ptr(out_codes)
        c.s_out_codes = float(s_out_codes)
        c.out_bits = int(out_bits)
    check("mkq_bert_layer", lib().mkq_bert_layer(
        ctypes.byref(c), _ptr(h_in), batch, max_seq, _ptr(cu_seqlens), T, _ptr(h_out), _ptr(ws), ws.numel(),
        _stream(stream)))
    return h_out
