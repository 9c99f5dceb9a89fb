"""CPU-only checks of the C-ABI boundary: the library loads, exports every
symbol include/mkq.h declares, and validates arguments (documented status
codes, nothing launched) without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2203_13483_b200 import _lib
from paper_2203_13483_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mkq.h")


@pytest.fixture(scope="module")
def L():
    B.build()
    return _lib.lib()


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"MKQ_API\s+[\w\s\*]*?\b(mkq_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported(L):
    names = declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert sorted(_lib.SIGNATURES) == names


def test_header_compiles_as_c():
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write('#include "mkq.h"\nint main(void){return mkq_version() > 0 ? 0 : 1;}\n')
        subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.dirname(HDR), "-c", c,
                               "-o", os.path.join(d, "t.o")])


def test_version_and_strings(L):
    assert L.mkq_version() == 10000
    assert L.mkq_status_string(0) == b"MKQ_OK"
    assert L.mkq_status_string(6) == b"MKQ_ERR_DEVICE"
    assert L.mkq_status_string(99) == b"MKQ_ERR_UNKNOWN"


FAKE = ctypes.c_void_p(0x10000)   # 16-byte aligned, never dereferenced on the host


def gemm(L, **kw):
    a = dict(a=FAKE, lda=384, w=FAKE, ldw=384, M=128, N=768, K=768, s_a=0.5, s_w=FAKE, bias=None,
             epi=None, out=FAKE, ldo=3072, ws=None, wsb=0, st=None)
    a.update(kw)
    return L.mkq_gemm_w4a4(*a.values())


def test_gemm_validation(L):
    assert gemm(L, a=None) == 1                      # NULL
    assert gemm(L, K=48) == 2                        # K % 32
    assert gemm(L, K=131072) == 2                    # K > MKQ_MAX_K
    assert gemm(L, N=40) == 2                        # N % 32
    assert gemm(L, lda=100) == 2                     # lda < K/2
    assert gemm(L, lda=392) == 3                     # lda % 16
    assert gemm(L, out=ctypes.c_void_p(0x10004)) == 3
    assert gemm(L, s_a=0.0) == 4                     # scale <= 0
    assert gemm(L, s_a=float("nan")) == 4
    assert gemm(L, s_a=float("inf")) == 4
    epi = _lib.MkqEpilogue(_lib.OUT_I4, 1, 0.1, -7, 8)   # literal [-7,8] range: 8 is not int4
    assert gemm(L, epi=ctypes.byref(epi), ldo=384) == 5
    epi = _lib.MkqEpilogue(_lib.OUT_I4, 1, -1.0, -8, 7)
    assert gemm(L, epi=ctypes.byref(epi), ldo=384) == 4
    epi = _lib.MkqEpilogue(9, 0, 1.0, 0, 0)
    assert gemm(L, epi=ctypes.byref(epi)) == 5
    assert gemm(L, M=0) == 0                         # empty: no-op
    assert b"K=" in L.mkq_last_error() or len(L.mkq_last_error()) >= 0


def test_valid_gemm_reports_device_error_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert gemm(L) == 6                               # MKQ_ERR_DEVICE, nothing launched


def test_quantize_and_glue_validation(L):
    q = L.mkq_quantize_pack
    assert q(None, 4, 32, 32, FAKE, 0, 4, -8, 7, FAKE, 16, None) == 1
    assert q(FAKE, 4, 31, 32, FAKE, 0, 4, -8, 7, FAKE, 16, None) == 2      # odd int4 cols
    assert q(FAKE, 4, 32, 32, FAKE, 0, 5, -8, 7, FAKE, 16, None) == 5      # bits
    assert q(FAKE, 4, 32, 32, FAKE, 0, 4, -7, 8, FAKE, 16, None) == 5      # [-7,8] not int4
    assert q(FAKE, 4, 32, 32, FAKE, 0, 8, -129, 127, FAKE, 32, None) == 5
    assert q(FAKE, 0, 32, 32, FAKE, 0, 4, -8, 7, FAKE, 16, None) == 0      # empty
    a = L.mkq_attention
    assert a(FAKE, 192, 1, 128, None, 128, 1, 32, 0, 1.0, -8, 7, FAKE, 256, None) == 2   # head_dim
    assert a(FAKE, 192, 1, 128, None, 100, 1, 64, 0, 1.0, -8, 7, FAKE, 256, None) == 2   # tokens
    assert a(FAKE, 192, 1, 128, None, 128, 1, 64, 3, 0.0, -8, 7, FAKE, 32, None) == 4    # s_out
    ln = L.mkq_residual_layernorm
    assert ln(FAKE, None, 4, 30, 32, FAKE, FAKE, 1e-12, FAKE, 0, 1.0, 0, 0, None, 0, None) == 2
    assert ln(FAKE, None, 4, 32, 32, FAKE, FAKE, 1e-12, FAKE, 4, 1.0, -8, 7, None, 16, None) == 1


def test_layer_validation(L):
    lay = _lib.MkqLayer()
    assert L.mkq_bert_layer(ctypes.byref(lay), FAKE, 1, 128, None, 128, FAKE, FAKE, 1 << 30, None) == 1
    for f in ("w_qkv", "w_o", "w_1", "w_2", "sw_qkv", "sw_o", "sw_1", "sw_2", "b_qkv", "b_o", "b_1", "b_2",
              "ln1_g", "ln1_b", "ln2_g", "ln2_b"):
        setattr(lay, f, 0x10000)
    lay.hidden, lay.heads, lay.ffn, lay.bits = 768, 12, 3072, 4
    lay.s_qkv_in = lay.s_o_in = lay.s_ffn1_in = lay.s_ffn2_in = 0.5
    lay.ln_eps = 1e-12
    need = L.mkq_bert_layer_workspace_size(ctypes.byref(lay), 128)
    assert need > 128 * 768 * 4
    assert L.mkq_bert_layer(ctypes.byref(lay), FAKE, 1, 128, None, 128, FAKE, FAKE, need - 1, None) == 7
    lay.heads = 11
    assert L.mkq_bert_layer(ctypes.byref(lay), FAKE, 1, 128, None, 128, FAKE, FAKE, need, None) == 2
    lay.heads = 12
    lay.bits = 2
    assert L.mkq_bert_layer(ctypes.byref(lay), FAKE, 1, 128, None, 128, FAKE, FAKE, need, None) == 5
    lay.bits = 4
    lay.s_o_in = -1.0
    assert L.mkq_bert_layer(ctypes.byref(lay), FAKE, 1, 128, None, 128, FAKE, FAKE, need, None) == 4
