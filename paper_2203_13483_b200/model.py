"""Layer assembly on top of the C ABI: offline weight prep (§8a-a0), offline
activation-scale calibration (★s host rule) and the
mixed-precision stack (P:243 'start from the last layer'; P:46 50% int4 +
50% int8).  Marshalling only: all arithmetic runs in libmkq.so kernels,
including the calibration statistic (mkq_act_scale)."""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import mkq as M


def act_range(bits: int):
    return (-8, 7) if bits == 4 else (-128, 127)


def weight_range(bits: int):
    return (-7, 7) if bits == 4 else (-127, 127)


def prepare_weight(w: torch.Tensor, bits: int):
    """a0: per-output-channel max-abs scale (R5/R6) and packed codes."""
    lo, hi = weight_range(bits)
    s_w = M.mkq_absmax_scale(w, float(hi), per_row=True)
    q = M.mkq_quantize_pack(w, s_w, bits, lo, hi, per_row=True)
    return q, s_w


def act_scale(x: torch.Tensor, l_max: int, p: float = 0.9999) -> float:
    """s_a = fl32(quantile_p(|x|)) / l_max (P:72 'top 0.01%', R6), computed
    on the GPU by mkq_act_scale (exact radix select); one scalar read back,
    because mkq_layer carries the static scales as host floats."""
    return float(M.mkq_act_scale(x.contiguous(), float(l_max), p).item())


def build_layer(params, bits: int, device="cuda", scales: Optional[Dict[str, float]] = None,
                ln_eps: float = 1e-12) -> M.QLayer:
    """params: synth.LayerFloat-like object with fp32 numpy/torch arrays."""
    def t(a):
        return torch.as_tensor(np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a).to(device)

    T = {}
    for name, wn, bn in (("qkv", "w_qkv", "b_qkv"), ("o", "w_o", "b_o"), ("1", "w_1", "b_1"), ("2", "w_2", "b_2")):
        q, s = prepare_weight(t(getattr(params, wn)).float(), bits)
        T["w_" + name] = q
        T["sw_" + name] = s
        T["b_" + name] = t(getattr(params, bn)).float()
    for n in ("ln1_g", "ln1_b", "ln2_g", "ln2_b"):
        T[n] = t(getattr(params, n)).float()
    sc = scales or {"s_qkv_in": 1.0, "s_o_in": 1.0, "s_ffn1_in": 1.0, "s_ffn2_in": 1.0}
    return M.QLayer(params.hidden, params.heads, params.ffn, bits, T, sc, ln_eps)


def calibrate(layer: M.QLayer, h: torch.Tensor, batch: int, max_seq: int,
              cu_seqlens: Optional[torch.Tensor] = None, int_attention: bool = False,
              trace: Optional[dict] = None) -> Dict[str, float]:
    """Sequential calibration of the static activation scales on a
    calibration batch, each quantization point in pipeline
    order with the scales already fixed upstream; returns and installs them.
    int_attention: also calibrate s_attn (p99.99 of |q|k|v| / 127) and run
    the NEXT(2) integer attention core (R19).  trace: if a dict is given, it
    receives the device tensor each scale was taken from (for the tests)."""
    bits, hd, F = layer.bits, layer.hidden, layer.ffn
    lo, hi = act_range(bits)
    t = layer.t
    gemm = M.mkq_gemm_w4a4 if bits == 4 else M.mkq_gemm_w8a8
    s = {}
    s["s_qkv_in"] = act_scale(h, hi)
    c = M.mkq_quantize_pack(h, torch.tensor([s["s_qkv_in"]], device=h.device), bits, lo, hi)
    if int_attention:
        qkv32 = gemm(c, t["w_qkv"], s["s_qkv_in"], t["sw_qkv"], t["b_qkv"], mode=M.OUT_F32, K=hd)
        s["s_attn"] = act_scale(qkv32, 127)
        qkv8 = gemm(c, t["w_qkv"], s["s_qkv_in"], t["sw_qkv"], t["b_qkv"], mode=M.OUT_I8, s_out=s["s_attn"],
                    qmin=-127, qmax=127, K=hd, requant_table=False)
        oa = M.mkq_attention_i8(qkv8, layer.heads, batch, max_seq, s["s_attn"], cu_seqlens, mode=M.OUT_F32)
    else:
        qkv = gemm(c, t["w_qkv"], s["s_qkv_in"], t["sw_qkv"], t["b_qkv"], mode=M.OUT_F16, K=hd)
        oa = M.mkq_attention(qkv, layer.heads, batch, max_seq, cu_seqlens, mode=M.OUT_F32)
    s["s_o_in"] = act_scale(oa, hi)
    c = M.mkq_quantize_pack(oa, torch.tensor([s["s_o_in"]], device=h.device), bits, lo, hi)
    o = gemm(c, t["w_o"], s["s_o_in"], t["sw_o"], t["b_o"], mode=M.OUT_F32, K=hd)
    h1 = M.mkq_residual_layernorm(o, h, t["ln1_g"], t["ln1_b"], layer.ln_eps)
    s["s_ffn1_in"] = act_scale(h1, hi)
    c = M.mkq_quantize_pack(h1, torch.tensor([s["s_ffn1_in"]], device=h.device), bits, lo, hi)
    g = gemm(c, t["w_1"], s["s_ffn1_in"], t["sw_1"], t["b_1"], mode=M.OUT_F32, gelu=True, K=hd)
    s["s_ffn2_in"] = act_scale(g, hi)
    if trace is not None:
        trace.update(h=h, qkv=qkv32 if int_attention else qkv, oa=oa, o=o, h1=h1, g=g)
    rebuilt = M.QLayer(hd, layer.heads, F, bits, layer.t, s, layer.ln_eps, use_table=layer.table is not None)
    layer.__dict__.update(rebuilt.__dict__)
    return s


def bit_plan(layers: int, n_int4: int) -> List[int]:
    """'we start from the last layer for quantization': the last
    n_int4 layers are W4A4, the rest W8A8 (Table 1 caption P:211)."""
    return [4 if i >= layers - n_int4 else 8 for i in range(layers)]


def compression_ratio(plan: Sequence[int]) -> float:
    """fp32 bits / mean weight bits (P:30 '5.3x of bits reduction')."""
    return 32.0 / (sum(plan) / len(plan))


class Encoder:
    """A stack of quantized BERT layers run back to back through
    mkq_bert_layer on one stream (CUDA-graph capturable).

    fuse_codes (NEXT(4) fused glue, default on): layer i's LN2 also writes
    layer i+1's input codes (Eq.1 with layer i+1's s_qkv_in and bits), so every
    layer after the first skips its input quantize pass; bit-identical to the
    unfused stack (tests/test_gpu_layer.py)."""

    def __init__(self, layers: List[M.QLayer], fuse_codes: bool = True):
        self.layers = layers
        self.fuse_codes = fuse_codes
        self._ws = None
        self._codes = None

    def __call__(self, h: torch.Tensor, batch: int, max_seq: int, cu_seqlens=None, stream=None,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Runs every layer in place on `out` (a copy of h unless given)."""
        T = h.shape[0]
        need = max(l.workspace_size(T) for l in self.layers)
        if self._ws is None or self._ws.numel() < need or self._ws.device != h.device:
            self._ws = torch.empty(need, dtype=torch.uint8, device=h.device)
        cb = max(l.hidden * l.bits // 8 for l in self.layers)
        if self.fuse_codes and (self._codes is None or self._codes.numel() < T * cb or self._codes.device != h.device):
            self._codes = torch.empty(T * cb, dtype=torch.uint8, device=h.device)
        cur = h
        n = len(self.layers)
        for i, l in enumerate(self.layers):
            kw = {}
            if self.fuse_codes:
                if i > 0:
                    kw["in_codes"] = self._codes
                if i + 1 < n:
                    nxt = self.layers[i + 1]
                    kw.update(out_codes=self._codes, s_out_codes=nxt.scales["s_qkv_in"], out_bits=nxt.bits)
            cur = M.mkq_bert_layer(l, cur, batch, max_seq, cu_seqlens, h_out=out, ws=self._ws, stream=stream, **kw)
            if out is None:
                out = cur
        return cur
