"""ctypes loader for libmkq.so (include/mkq.h).  Fails loudly: there is no
CPU or eager fallback for any entry point."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("MKQ_LIB") or os.path.join(HERE, "libmkq.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
F32 = ctypes.c_float
SZ = ctypes.c_size_t

OK = 0
STATUS = {0: "MKQ_OK", 1: "MKQ_ERR_NULL", 2: "MKQ_ERR_SHAPE", 3: "MKQ_ERR_ALIGN", 4: "MKQ_ERR_SCALE",
          5: "MKQ_ERR_RANGE", 6: "MKQ_ERR_DEVICE", 7: "MKQ_ERR_WORKSPACE", 8: "MKQ_ERR_CUDA"}

OUT_F32, OUT_BF16, OUT_I32, OUT_I4, OUT_I8, OUT_F16 = 0, 1, 2, 3, 4, 5

# Every symbol include/mkq.h declares, with its ctypes signature.
SIGNATURES = {
    "mkq_status_string": (ctypes.c_char_p, [I32]),
    "mkq_last_error": (ctypes.c_char_p, []),
    "mkq_version": (I32, []),
    "mkq_quantize_pack": (I32, [P, I64, I64, I64, P, I32, I32, I32, I32, P, I64, P]),
    "mkq_absmax_scale": (I32, [P, I64, I64, I64, I32, F32, P, P]),
    "mkq_gemm_w4a4": (I32, [P, I64, P, I64, I64, I64, I64, F32, P, P, P, P, I64, P, SZ, P]),
    "mkq_gemm_w8a8": (I32, [P, I64, P, I64, I64, I64, I64, F32, P, P, P, P, I64, P, SZ, P]),
    "mkq_gemm_workspace_size": (SZ, [I64, I64, I64]),
    "mkq_gemm_residual_ln_workspace_size": (SZ, [I64, I64]),
    "mkq_gemm_residual_ln": (I32, [P, I64, P, I64, I64, I64, I64, F32, P, P, P, I64, P, P, F32, P, I64, I32, F32,
                                   I32, I32, P, I64, P, SZ, P]),
    "mkq_gemm_gather_arrivals": (I32, [I64, I64]),
    "mkq_gemm_w4a4_gather": (I32, [P, I64, P, I64, I64, I64, I64, F32, P, P, P, P, I32, I64, I64, P, P]),
    "mkq_wait_counter": (I32, [P, ctypes.c_uint32, P]),
    "mkq_ipc_get_handle": (I32, [P, P, P]),
    "mkq_ipc_open_handle": (I32, [P, P]),
    "mkq_ipc_close": (I32, [P]),
    "mkq_set_small_m_mode": (None, [I32]),
    "mkq_requant_table_size": (SZ, []),
    "mkq_requant_table": (I32, [I32, F32, I32, I32, P, SZ, P]),
    "mkq_attention": (I32, [P, I64, I64, I64, P, I64, I32, I32, I32, F32, I32, I32, P, I64, P]),
    "mkq_attention_i8": (I32, [P, I64, I64, I64, P, I64, I32, I32, F32, I32, F32, I32, I32, P, I64, P]),
    "mkq_residual_layernorm": (I32, [P, P, I64, I64, I64, P, P, F32, P, I32, F32, I32, I32, P, I64, P]),
    "mkq_interleave_blocks": (I32, [P, P, I64, I64, I64, I64, P]),
    "mkq_fake_quant_workspace_size": (SZ, [I64]),
    "mkq_fake_quant": (I32, [P, I64, P, I32, I32, P, P, P, P, P, SZ, P]),
    "mkq_act_scale_workspace_size": (SZ, []),
    "mkq_act_scale": (I32, [P, I64, ctypes.c_double, F32, P, P, SZ, P]),
    "mkq_bert_layer_workspace_size": (SZ, [P, I64]),
    "mkq_layer_fused_ln": (I32, [P, I64]),
    "mkq_bert_layer": (I32, [P, P, I64, I64, P, I64, P, P, SZ, P]),
}


class MkqEpilogue(ctypes.Structure):
    _fields_ = [("out", ctypes.c_int32), ("gelu", ctypes.c_int32), ("s_out", ctypes.c_float),
                ("qmin_out", ctypes.c_int32), ("qmax_out", ctypes.c_int32), ("requant_table", ctypes.c_void_p)]


class MkqLayer(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("heads", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("bits", ctypes.c_int32)] + \
        [(n, ctypes.c_void_p) for n in ("w_qkv", "w_o", "w_1", "w_2", "sw_qkv", "sw_o", "sw_1", "sw_2",
                                        "b_qkv", "b_o", "b_1", "b_2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")] + \
        [(n, ctypes.c_float) for n in ("s_qkv_in", "s_o_in", "s_ffn1_in", "s_ffn2_in", "ln_eps")] + \
        [("ffn1_requant_table", ctypes.c_void_p), ("int_attention", ctypes.c_int32), ("s_attn", ctypes.c_float),
         ("in_codes", ctypes.c_void_p), ("out_codes", ctypes.c_void_p), ("s_out_codes", ctypes.c_float),
         ("out_bits", ctypes.c_int32)]


class MkqError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(
                f"libmkq.so not found at {SO}: build it with `python -m paper_2203_13483_b200.build` "
                "(there is no fallback implementation)")
        L = ctypes.CDLL(SO)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("MKQ_LIB") and not hasattr(L, name):
                continue   # diagnostics: an older build selected with MKQ_LIB may lack newer entry points
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(fn: str, status: int):
    if status != OK:
        raise MkqError(fn, status, lib().mkq_last_error().decode(errors="replace"))
