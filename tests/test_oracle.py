"""Pins of the CPU oracle against what the paper and the mathematics fix
(never against the oracle itself).  CPU-only (-m "not gpu")."""
import csv
import math
import os

import numpy as np
import pytest
from scipy.special import erf

import oracle
from oracle import layer as OL
import synth
from tests.exact import dequant_exact, quant_exact, rn32, f32

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return list(csv.DictReader(line for line in f if not line.startswith("#")))


# ---------------------------------------------------------------- quantizer
def test_paper_worked_example_P145_149():
    """x=(0.2,0.9), s=1 -> Q=(0,1); s=0.9 -> Q=(0,0.9)."""
    x = np.array([[0.2, 0.9]], np.float32)
    assert oracle.quantize(x, 1.0, -8, 7).tolist() == [[0, 1]]
    assert oracle.fake_quant(x, 1.0, -8, 7).tolist() == [0.0, 1.0]
    q = oracle.fake_quant(x, 0.9, -8, 7)
    assert q[0] == 0.0 and q[1] == np.float32(0.9)


def test_paper_scale_gradients_P151_P187():
    """STE gradient -0.1 and MSE gradient +0.2."""
    x = np.array([0.2, 0.9], np.float32)
    assert oracle.scale_grad_ste(x, 1.0) == pytest.approx(-0.1, abs=1e-7)
    assert oracle.scale_grad_mse(x, 1.0) == pytest.approx(0.2, abs=1e-7)
    # "if we decrease s into 0.9 ... a better quantization choice":
    mse = lambda s: float(np.sum((oracle.fake_quant(x, s, -8, 7).astype(np.float64)
                                  - x.astype(np.float64)) ** 2))
    assert mse(0.9) == pytest.approx(0.04, abs=1e-6)
    assert mse(1.0) == pytest.approx(0.05, abs=1e-6)
    assert mse(0.9) < mse(1.0)


def test_qat_gradients_hand_worked_with_clipping():
    """x=(0.2,0.9,-0.3,7.6,-9.0), s=1, codes [-8,7] (worked by hand):
    unclamped codes (0,1,0,8,-9) -> the last two are clipped (R18).
    STE (P:138-142 + LSQ rule for clipped, R17): (-0.2+0)+(-0.9+1)+(0.3+0)+7-8 = -0.8.
    MSE: 2[(0-.2)0 + (1-.9)1 + (0+.3)0 + (7-7.6)7 + (-8+9)(-8)] = -24.2.
    STE input gradient: grad_y passes where not clipped -> (1,2,3,0,0)."""
    x = np.array([0.2, 0.9, -0.3, 7.6, -9.0], np.float32)
    assert oracle.scale_grad_ste(x, 1.0) == pytest.approx(-0.8, abs=1e-6)
    assert oracle.scale_grad_mse(x, 1.0) == pytest.approx(-24.2, abs=1e-5)
    gx = oracle.ste_grad_x(x, np.array([1, 2, 3, 4, 5], np.float32), 1.0)
    assert gx.tolist() == [1.0, 2.0, 3.0, 0.0, 0.0]
    # a code that rounds onto the bound is not clipped: 7.4 -> 7, -8.4 -> -8
    y = np.array([7.4, -8.4], np.float32)
    assert oracle.ste_grad_x(y, np.ones(2, np.float32), 1.0).tolist() == [1.0, 1.0]


def test_qat_gradients_match_torch_lsq():
    """Library pin: PyTorch's LSQ fake-quant (esser2019learned, the 'previous
    work' of P:128) with grad_factor 1 and dL/dQ = 1 gives d/ds = the STE
    scale gradient and d/dx = the STE input mask.  Inputs are kept away from
    rounding boundaries, where torch's x*(1/s) and Eq.1's x/s (R3) agree."""
    import torch
    rng = np.random.default_rng(21)
    s = np.float32(0.37)
    x = (rng.standard_normal(20000) * 1.5).astype(np.float32)
    v = x.astype(np.float64) / np.float64(s)
    x = x[np.abs(np.abs(v - np.floor(v)) - 0.5) > 1e-3]
    xt = torch.from_numpy(x.copy()).requires_grad_(True)
    st = torch.tensor([float(s)], requires_grad=True)
    y = torch._fake_quantize_learnable_per_tensor_affine(xt, st, torch.tensor([0.0]), -8, 7, 1.0)
    y.backward(torch.ones_like(y))
    assert np.array_equal(y.detach().numpy(), oracle.fake_quant(x, s, -8, 7))
    assert np.array_equal(xt.grad.numpy(), oracle.ste_grad_x(x, np.ones_like(x), s))
    assert (~(xt.grad.numpy() > 0)).sum() > 10          # some clipped elements exercised
    g = oracle.scale_grad_ste(x, s)
    assert float(st.grad) == pytest.approx(g, rel=1e-4, abs=1e-2)


def test_mse_gradient_matches_finite_difference():
    """§4.1.2: away from rounding ties the MSE gradient is the
    derivative of sum (Q[x]-x)^2 w.r.t. s (codes fixed under a small ds)."""
    rng = np.random.default_rng(3)
    x = rng.uniform(-3, 3, 2000).astype(np.float32)
    s = 0.37
    v = x.astype(np.float64) / s
    keep = np.abs(v - np.round(v)) < 0.45       # away from ties
    x = x[keep]
    h = 1e-7
    codes = np.clip(np.rint(x.astype(np.float64) / s), -8, 7)
    f = lambda ss: np.sum((ss * codes - x.astype(np.float64)) ** 2)
    fd = (f(s + h) - f(s - h)) / (2 * h)
    assert oracle.scale_grad_mse(x, s) == pytest.approx(fd, rel=1e-4)


def test_quantizer_golden_table():
    for r in _rows("quantizer_table.csv"):
        x, s = np.float32(float(r["x"])), np.float32(float(r["s"]))
        got = int(oracle.quantize(np.array([[x]], np.float32), s, -8, 7)[0, 0])
        assert got == int(r["code"]), r
        assert got == quant_exact(x, s, -8, 7), r


def test_quantizer_exact_rational_bruteforce():
    rng = np.random.default_rng(11)
    xs = synth.activations(1, 4000, seed=5)[0]
    xs = np.concatenate([xs, rng.integers(-20, 20, 500).astype(np.float32) + np.float32(0.5),
                         np.float32([0.0, -0.0, 1e-30, -1e-30, 3e38, -3e38])])
    for s in [np.float32(0.1), np.float32(0.3), np.float32(0.5558), np.float32(1.0),
              np.float32(0.0123)]:
        q = oracle.quantize(xs[None, :], s, -8, 7)[0]
        for x, c in zip(xs[::7], q[::7]):
            assert int(c) == quant_exact(x, s, -8, 7), (x, s)
        q8 = oracle.quantize(xs[None, :], s, -128, 127)[0]
        for x, c in zip(xs[::13], q8[::13]):
            assert int(c) == quant_exact(x, s, -128, 127), (x, s)


def test_quantizer_invariants_1e6():
    x = synth.activations(1000, 1000, seed=1)
    s = np.float32(0.5558)
    q = oracle.quantize(x, s, -8, 7)
    assert q.min() >= -8 and q.max() <= 7
    v = x.astype(np.float64) / float(s)
    unclipped = (v >= -8.5) & (v <= 7.5)
    err = np.abs(x.astype(np.float64) - float(s) * q.astype(np.float64))
    assert np.all(err[unclipped] <= float(s) / 2 * (1 + 2.0 ** -22))
    # idempotence on lattice points s*q (exact in fp32 for |q| <= 8 here)
    lat = (np.float32(s) * q.astype(np.float32))
    assert np.array_equal(oracle.quantize(lat, s, -8, 7), q)
    # weights range [-7,7]
    qw = oracle.quantize(x, s, -7, 7)
    assert np.abs(qw).max() <= 7
    assert oracle.quantize(np.float32([[0.0, -0.0]]), s, -8, 7).tolist() == [[0, 0]]


def test_per_row_scale():
    x = synth.activations(8, 64, seed=2)
    s = np.linspace(0.1, 1.0, 8).astype(np.float32)
    q = oracle.quantize(x, s, -8, 7, per_row=True)
    for i in range(8):
        assert np.array_equal(q[i], oracle.quantize(x[i:i + 1], s[i], -8, 7)[0])


# ---------------------------------------------------------------- packing
def test_pack_hand_bytes():
    for r in _rows("pack_bytes.csv"):
        p = oracle.pack_int4(np.array([[int(r["lo"]), int(r["hi"])]], np.int8))
        assert int(p[0, 0]) == int(r["byte"], 16), r


def test_unpack_pack_all_bytes():
    b = np.arange(256, dtype=np.uint8)[None, :]
    q = oracle.unpack_int4(b, 512)
    assert q.min() == -8 and q.max() == 7
    assert np.array_equal(oracle.pack_int4(q), b)
    # nibble semantics written out: low nibble = even element
    for v in [0x00, 0x0F, 0xF0, 0x78, 0x87, 0x53]:
        lo, hi = v & 0xF, v >> 4
        sx = lambda n: n - 16 if n >= 8 else n
        assert q[0, 2 * v] == sx(lo) and q[0, 2 * v + 1] == sx(hi)


# ---------------------------------------------------------------- GEMM
def test_gemm_hand_case():
    A = np.array([[1, -8], [7, 0]], np.int8)
    W = np.array([[-7, 7], [2, 3]], np.int8)
    assert oracle.gemm_i32(A, W).tolist() == [[-63, -22], [-49, 14]]


def test_gemm_vs_int64_matmul():
    rng = np.random.default_rng(0)
    for (M, N, K) in [(1, 1, 1), (3, 5, 7), (17, 33, 64), (64, 32, 256)]:
        A = rng.integers(-8, 8, (M, K)).astype(np.int8)
        W = rng.integers(-7, 8, (N, K)).astype(np.int8)
        ref = A.astype(np.int64) @ W.astype(np.int64).T
        assert np.array_equal(oracle.gemm_i32(A, W), ref)


def test_gemm_zero_padding_and_worst_case():
    rng = np.random.default_rng(1)
    A = rng.integers(-8, 8, (5, 32)).astype(np.int8)
    W = rng.integers(-7, 8, (6, 32)).astype(np.int8)
    Ap = np.concatenate([A, np.zeros((5, 32), np.int8)], 1)
    Wp = np.concatenate([W, rng.integers(-7, 8, (6, 32)).astype(np.int8)], 1)
    assert np.array_equal(oracle.gemm_i32(A, W), oracle.gemm_i32(Ap, Wp))
    K = 4096
    assert oracle.gemm_i32(np.full((1, K), -8, np.int8), np.full((1, K), -7, np.int8))[0, 0] == 229376
    assert oracle.gemm_i32(np.full((1, K), -8, np.int8), np.full((1, K), 7, np.int8))[0, 0] == -229376
    assert oracle.gemm_i32(np.full((1, K), -128, np.int8),
                           np.full((1, K), -127, np.int8))[0, 0] == 66584576
    with pytest.raises(RuntimeError):  # exceeds int32: detected, not wrapped
        oracle.gemm_i32(np.full((1, 140000), -128, np.int8), np.full((1, 140000), -127, np.int8))


def test_w8a8_equals_w4a4_when_codes_fit():
    rng = np.random.default_rng(2)
    A = rng.integers(-8, 8, (9, 96)).astype(np.int8)
    W = rng.integers(-7, 8, (11, 96)).astype(np.int8)
    # through the int4 packing round trip and straight int8
    A4 = oracle.unpack_int4(oracle.pack_int4(A), 96)
    assert np.array_equal(oracle.gemm_i32(A4, W), oracle.gemm_i32(A, W))


# ---------------------------------------------------------------- dequant
def test_dequant_exact_rational():
    rng = np.random.default_rng(4)
    acc = rng.integers(-229376, 229377, (7, 13)).astype(np.int32)
    acc[0, :] = 0
    s_a = np.float32(0.5558)
    s_w = rng.uniform(1e-4, 1e-2, 13).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 13).astype(np.float32)
    y = oracle.dequant(acc, s_a, s_w, b)
    yn = oracle.dequant(acc, s_a, s_w, None)
    for m in range(7):
        for n in range(13):
            assert y[m, n] == dequant_exact(acc[m, n], s_a, s_w[n], b[n])
            assert yn[m, n] == dequant_exact(acc[m, n], s_a, s_w[n])
    assert np.array_equal(y[0], b)                          # acc = 0 -> bias
    one = np.ones(13, np.float32)
    assert np.array_equal(oracle.dequant(acc, 1.0, one, None), acc.astype(np.float32))


def test_dequant_equals_fake_quant_gemm_fp64():
    """Dequant == (s_a qa)(s_w qw)^T + b in fp64 within 2 ulp (S:520 idea)."""
    rng = np.random.default_rng(5)
    A = rng.integers(-8, 8, (16, 128)).astype(np.int8)
    W = rng.integers(-7, 8, (24, 128)).astype(np.int8)
    s_a = np.float32(0.31)
    s_w = rng.uniform(1e-3, 1e-2, 24).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 24).astype(np.float32)
    y = oracle.dequant(oracle.gemm_i32(A, W), s_a, s_w, b).astype(np.float64)
    ref = (float(s_a) * A.astype(np.float64)) @ (s_w.astype(np.float64)[:, None]
                                                  * W.astype(np.float64)).T + b
    # sc = fl(s_a*s_w) carries a relative error <= 2^-24 of the product term,
    # y carries one rounding of its own: bound by 2 ulp of the larger of |y|
    # and |acc*s_a*s_w| (cancellation against the bias).
    prod = np.abs(ref - b)
    ulp = np.spacing(np.maximum(np.abs(ref), prod).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(y - ref) <= 2 * ulp)


# ---------------------------------------------------------------- GELU
def test_gelu_closed_form_values():
    for r in _rows("gelu_values.csv"):
        y = float(r["y"])
        assert oracle.gelu_pinned(np.float32([y]))[0] == pytest.approx(float(r["gelu"]), abs=2e-6)


def test_gelu_dense_grid_vs_fp64_erf():
    y = np.concatenate([np.linspace(-16, 16, 2_000_001, dtype=np.float32),
                        np.logspace(-6, 0, 200_001).astype(np.float32),
                        -np.logspace(-6, 0, 200_001).astype(np.float32)])
    g = oracle.gelu_pinned(y).astype(np.float64)
    yd = y.astype(np.float64)
    ref = 0.5 * yd * (1.0 + erf(yd / math.sqrt(2.0)))
    assert np.all(np.abs(g - ref) <= 1e-6 * np.maximum(1.0, np.abs(yd)))
    assert oracle.gelu_pinned(np.float32([0.0]))[0] == 0.0
    big = np.float32([6.0, 20.0, 1e6])
    assert np.array_equal(oracle.gelu_pinned(big), big)          # erf -> 1
    assert np.all(oracle.gelu_pinned(-big) == 0.0)


def test_erf_pinned_odd_pieces():
    for t in [0.0, 0.5, 0.999, 1.0, 2.5, 3.91, 3.92, 5.0]:
        assert abs(oracle.erf_pinned(t) - math.erf(t)) < 2e-7


# ---------------------------------------------------------------- conversions
def test_f16_bf16_rounding():
    import torch
    rng = np.random.default_rng(6)
    x = np.concatenate([rng.standard_normal(3000).astype(np.float32) * 100,
                        np.float32([0, -0.0, 65504, 65519.99, 65520, 1e-8, 6e-5, 1e30, -1e30]),
                        rng.standard_normal(1000).astype(np.float32) * 1e-6])
    assert np.array_equal(oracle.f32_to_f16_bits(x), x.astype(np.float16).view(np.uint16))
    bf = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(oracle.f32_to_bf16_bits(x), bf)


# ---------------------------------------------------------------- linear composition
def test_linear_modes_compose():
    rng = np.random.default_rng(8)
    A = rng.integers(-8, 8, (6, 64)).astype(np.int8)
    W = rng.integers(-7, 8, (10, 64)).astype(np.int8)
    s_a, s_w = np.float32(0.5), rng.uniform(1e-2, 5e-2, 10).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 10).astype(np.float32)
    acc = A.astype(np.int64) @ W.astype(np.int64).T        # library routine
    assert np.array_equal(oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_I32), acc)
    y = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_F32)
    for m in range(6):
        for n in range(10):
            assert y[m, n] == dequant_exact(int(acc[m, n]), s_a, s_w[n], b[n])
    g = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_F32, gelu=True)
    s_out = np.float32(0.07)
    q = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_I4, gelu=True, s_out=s_out)
    for m in range(6):
        for n in range(10):
            assert q[m, n] == quant_exact(g[m, n], s_out, -8, 7)
    h = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_F16)
    assert np.array_equal(h, y.astype(np.float16).view(np.uint16))


# ---------------------------------------------------------------- calibration
def test_absmax_weight_scale():
    w = synth.weight(64, 256, seed=9)
    s = oracle.absmax_scale(w, 7)
    q = oracle.quantize(w, s, -7, 7, per_row=True)
    assert np.all(np.abs(q).max(axis=1) == 7)      # max-abs element -> +-7
    for i in range(64):
        assert s[i] == np.float32(np.abs(w[i]).max()) / np.float32(7)
    z = np.zeros((2, 8), np.float32)
    assert np.all(oracle.absmax_scale(z, 7) == np.float32(1e-8))
    assert np.all(oracle.absmax_scale(w * np.float32(4), 7) == s * np.float32(4))


def test_activation_quantile_half_normal():
    x = np.random.default_rng(10).standard_normal(1_000_000)
    q = oracle.abs_quantile(x, 0.9999)
    assert abs(q - 3.8906) < 0.06       # half-normal 0.9999 quantile
    assert oracle.abs_quantile(np.ones(100), 0.9999) == 1.0
    # hand cases: |x| sorted = (1,2,3,4); p=0.5 -> pos 1.5 -> 2.5; p=0 -> min, p=1 -> max
    t = np.array([3, -1, 2, -4], np.float32)
    assert oracle.abs_quantile(t, 0.5) == np.float32(2.5)
    assert oracle.abs_quantile(t, 0.0) == np.float32(1.0)
    assert oracle.abs_quantile(t, 1.0) == np.float32(4.0)
    # library pin: numpy's linear-interpolation quantile (same definition)
    u = np.random.default_rng(11).standard_normal(100_003).astype(np.float32)
    for p in (0.9999, 0.5, 0.123456):
        ref = np.quantile(np.abs(u.astype(np.float64)), p, method="linear")
        assert oracle.abs_quantile(u, p) == pytest.approx(ref, rel=2e-7)


def test_bit_accounting_P30():
    """5.3x bits reduction for 50% int4 + 50% int8 layers."""
    assert 32 / ((4 + 8) / 2) == pytest.approx(5.333, abs=1e-3)
    q = np.zeros((4, 64), np.int8)
    assert oracle.pack_int4(q).nbytes * 8 == np.zeros((4, 64), np.float32).nbytes


# ---------------------------------------------------------------- layer glue
def test_softmax_layernorm_closed_forms():
    x = np.random.default_rng(12).standard_normal((5, 37)) * 30
    p = OL.softmax(x)
    assert np.allclose(p.sum(-1), 1.0, atol=1e-12)
    y = OL.layernorm(x, np.ones(37), np.zeros(37))
    assert np.allclose(y.mean(-1), 0, atol=1e-12)
    assert np.allclose(y.var(-1), 1, atol=1e-9)
    assert np.allclose(OL.softmax(np.zeros((2, 4))), 0.25)


def test_attention_bruteforce_and_uniform():
    rng = np.random.default_rng(13)
    d, heads, L = 8, 2, 5
    qkv = rng.standard_normal((2 * L, 3 * d))
    out = OL.attention(qkv, [L, L], heads)
    dk = d // heads
    for b in range(2):
        for a in range(heads):
            for i in range(L):
                r = b * L + i
                q = qkv[r, a * dk:(a + 1) * dk]
                sc = [sum(q[t] * qkv[b * L + j, d + a * dk + t] for t in range(dk)) / math.sqrt(dk)
                      for j in range(L)]
                mx = max(sc)
                e = [math.exp(v - mx) for v in sc]
                Z = sum(e)
                for t in range(dk):
                    ref = sum(e[j] / Z * qkv[b * L + j, 2 * d + a * dk + t] for j in range(L))
                    assert out[r, a * dk + t] == pytest.approx(ref, abs=1e-12)
    # identical keys -> uniform attention -> mean of v (Eq.4-5)
    qkv2 = qkv.copy()
    qkv2[:L, d:2 * d] = qkv2[0, d:2 * d]
    out2 = OL.attention(qkv2, [L, L], heads)
    assert np.allclose(out2[:L], qkv2[:L, 2 * d:].mean(0, keepdims=True), atol=1e-12)


def test_layer_oracle_small_runs_and_is_consistent():
    p = synth.layer_params(64, 4, 128)
    W = OL.LayerWeights(64, 4, 128, 4,
                        OL.prepare_weight(p.w_qkv, p.b_qkv, 4), OL.prepare_weight(p.w_o, p.b_o, 4),
                        OL.prepare_weight(p.w_1, p.b_1, 4), OL.prepare_weight(p.w_2, p.b_2, 4),
                        p.ln1_g, p.ln1_b, p.ln2_g, p.ln2_b)
    h = synth.hidden_states(2, 16, 64, seed=3)
    OL.calibrate(synth.hidden_states(2, 16, 64, seed=1000000), W, [16, 16])
    T = OL.bert_layer(h, W, [16, 16])
    assert T.h_out.shape == (32, 64)
    assert np.allclose(T.h_out.astype(np.float64).mean(-1), (p.ln2_b.mean()), atol=0.05)
    assert T.codes_ffn2_in.min() >= -8 and T.codes_ffn2_in.max() <= 7
    # the quantized layer tracks the fp32 layer (QAT's premise): loose check
    assert np.isfinite(T.h_out).all()


# ---------------------------------------------------------------- NEXT(2) integer attention (R19)
def _codes_qkv(rng, L, heads=1, lim=127):
    return rng.integers(-lim, lim + 1, (L, 3 * 64 * heads)).astype(np.int8)


def test_int_attention_single_token_is_v():
    """L = 1: softmax of one score is 1 -> p = 255, OA = s * v exactly."""
    rng = np.random.default_rng(0)
    c = _codes_qkv(rng, 1, 2)
    s = np.float32(0.031)
    oa = OL.attention_int8(c, [1], 2, s)
    assert np.array_equal(oa, (c[:, 256:].astype(np.float32) * s).astype(np.float32))


def test_int_attention_equal_keys_is_mean_and_dominant_key_is_one_hot():
    rng = np.random.default_rng(1)
    s = np.float32(0.05)
    L = 17
    c = _codes_qkv(rng, L)
    c[:, 64:128] = c[0, 64:128]                  # identical keys -> all p = 255
    oa = OL.attention_int8(c, [L], 1, s)
    v = c[:, 128:].astype(np.int64)
    mean = (np.float32(255 * v.sum(0)) / np.float32(255 * L)).astype(np.float32)
    assert np.array_equal(oa[0], (mean * s).astype(np.float32))
    # one key aligned with every query, the rest zero: c*d = 0.0025*127*127*64/8 ~ 322 >> ln(254)
    c2 = np.zeros((L, 192), np.int8)
    c2[:, :64] = 127
    c2[5, 64:128] = 127
    c2[:, 128:] = _codes_qkv(rng, L)[:, 128:]
    oa2 = OL.attention_int8(c2, [L], 1, s)
    assert np.array_equal(oa2, np.tile((c2[5, 128:].astype(np.float32) * s).astype(np.float32), (L, 1)))


def test_int_attention_close_to_float_softmax():
    """Against the fp64 softmax of c*S on the dequantized v: each p_ij is
    255 e_ij rounded (error <= 1/2) and sum p >= 255, so
    |OA_int - OA| <= s max|v| L / 255."""
    rng = np.random.default_rng(2)
    s = np.float32(0.02)
    for L in (3, 40, 128):
        c = _codes_qkv(rng, L)
        oa = OL.attention_int8(c, [L], 1, s).astype(np.float64)
        q, k, v = (c[:, i * 64:(i + 1) * 64].astype(np.float64) for i in range(3))
        cc = float(np.float32(np.float32(s * s) * np.float32(0.125)))
        ref = OL.softmax(cc * (q @ k.T)) @ (v * float(s))
        bound = float(s) * np.abs(v).max() * L / 255
        assert np.abs(oa - ref).max() <= bound


def test_int_attention_bruteforce_tiny():
    """Per-element loop with Python ints and math.exp (independent of numpy's
    vectorized path) on a tiny case."""
    import math
    rng = np.random.default_rng(3)
    s = np.float32(0.04)
    L = 5
    c = _codes_qkv(rng, L, lim=20)
    oa = OL.attention_int8(c, [L], 1, s)
    cc = float(np.float32(np.float32(s * s) * np.float32(0.125)))
    for i in range(L):
        S = [sum(int(c[i, t]) * int(c[j, 64 + t]) for t in range(64)) for j in range(L)]
        p = [int(round(255 * math.exp(-cc * (max(S) - S[j])))) for j in range(L)]   # no exact ties here
        for t in range(64):
            num = sum(p[j] * int(c[j, 128 + t]) for j in range(L))
            y = np.float32(np.float32(num) / np.float32(sum(p)))
            assert oa[i, t] == np.float32(y * s)


# ---------------------------------------------------------------- layer composition and calibration pins
def _ln_textbook(x, g, b, eps=1e-12):
    """Row LayerNorm written out with math.fsum (independent of numpy's
    reductions): (x - mean) / sqrt(var + eps) * g + b (R9)."""
    out = np.empty(x.shape, dtype=np.float64)
    for r in range(x.shape[0]):
        row = [float(v) for v in x[r]]
        n = len(row)
        mu = math.fsum(row) / n
        var = math.fsum((v - mu) ** 2 for v in row) / n
        out[r] = [(v - mu) / math.sqrt(var + eps) * float(gg) + float(bb) for v, gg, bb in zip(row, g, b)]
    return out


def _zero_weight_layer(hidden=128, heads=2, ffn=256, bits=4, v_identity=False):
    """A layer whose weights are all zero (codes 0, s_w = 1e-8 floor) and whose
    biases / LN parameters are distinct random vectors: every Linear then
    returns its bias exactly (acc = 0 -> fma(0, sc, b) = b, R4), so each
    intermediate of Eq.2-5 / P:93-98 has a closed form.  v_identity: W^V =
    0.5 I instead (codes +-7 on the diagonal), so v carries the input."""
    rng = np.random.default_rng(77)
    z = lambda n, k: np.zeros((n, k), np.float32)  # noqa: E731
    b = lambda n, a: rng.uniform(-a, a, n).astype(np.float32)  # noqa: E731
    w_qkv = z(3 * hidden, hidden)
    if v_identity:
        w_qkv[2 * hidden:] = 0.5 * np.eye(hidden, dtype=np.float32)
    W = OL.LayerWeights(hidden, heads, ffn, bits,
                        OL.prepare_weight(w_qkv, b(3 * hidden, 1.0), bits),
                        OL.prepare_weight(z(hidden, hidden), b(hidden, 1.0), bits),
                        OL.prepare_weight(z(ffn, hidden), b(ffn, 3.0), bits),
                        OL.prepare_weight(z(hidden, ffn), b(hidden, 1.0), bits),
                        (1 + 0.3 * rng.standard_normal(hidden)).astype(np.float32), b(hidden, 0.5),
                        (1 + 0.3 * rng.standard_normal(hidden)).astype(np.float32), b(hidden, 0.5))
    return W


def test_layer_composition_closed_form_zero_weights():
    """bert_layer's composition (R8/R9) on a layer with zero weights:
    q|k|v = b^{QKV}; equal keys -> OA = b^V (Eq.4-5); o = b^A; h1 = LN1(b^A + h);
    the FFN2 input codes = Q(GELU(b^1)) (a5, a6); f = b^2; out = LN2(b^2 + h1).
    A swapped residual (h instead of h1), a dropped bias, LN1/LN2 parameters
    exchanged or the requant taken before GELU each fail one assertion."""
    W = _zero_weight_layer()
    W.s_qkv_in, W.s_o_in, W.s_ffn1_in, W.s_ffn2_in = (np.float32(v) for v in (0.5, 0.1, 0.4, 0.05))
    seqlens = [5, 11]
    M, d = sum(seqlens), W.hidden
    h = synth.hidden_states(1, M, d, seed=21)
    T = OL.bert_layer(h, W, seqlens)
    bq = W.qkv.bias
    assert np.array_equal(T.qkv, np.tile(bq, (M, 1)))
    assert np.allclose(T.oa, np.tile(bq[2 * d:], (M, 1)), rtol=1e-6, atol=0)
    assert np.array_equal(T.o, np.tile(W.o.bias, (M, 1)))
    h1 = _ln_textbook(T.o.astype(np.float64) + h, W.ln1_g, W.ln1_b)
    assert np.allclose(T.h1, h1, rtol=0, atol=2e-6)
    codes = oracle.quantize(oracle.gelu_pinned(W.w1.bias)[None, :], W.s_ffn2_in, -8, 7)
    assert np.array_equal(T.codes_ffn2_in, np.tile(codes, (M, 1)))
    assert np.array_equal(T.f, np.tile(W.w2.bias, (M, 1)))
    out = _ln_textbook(T.f.astype(np.float64) + T.h1, W.ln2_g, W.ln2_b)
    assert np.allclose(T.h_out, out, rtol=0, atol=2e-6)
    # the closed form separates the plausible mis-compositions
    wrong = _ln_textbook(T.f.astype(np.float64) + h, W.ln2_g, W.ln2_b)
    assert np.abs(wrong - out).max() > 1e-2


def test_layer_attention_pools_v_within_each_sequence():
    """With W^Q = W^K = 0 every query sees equal scores, so OA is the mean of
    the v rows of its own sequence (Eq.4-5, R13 sequence boundaries); W^V =
    0.5 I makes the v rows carry the (row-distinct) quantized input."""
    W = _zero_weight_layer(v_identity=True)
    W.s_qkv_in, W.s_o_in, W.s_ffn1_in, W.s_ffn2_in = (np.float32(v) for v in (0.5, 0.1, 0.4, 0.05))
    seqlens = [3, 1, 12]
    M, d = sum(seqlens), W.hidden
    h = synth.hidden_states(1, M, d, seed=22)
    T = OL.bert_layer(h, W, seqlens)
    v = T.qkv[:, 2 * d:].astype(np.float64)
    assert np.abs(v - v[0]).max() > 0.1           # rows differ: pooling is observable
    r0 = 0
    for L in seqlens:
        ref = v[r0:r0 + L].mean(axis=0)
        assert np.allclose(T.oa[r0:r0 + L], np.tile(ref, (L, 1)), rtol=1e-6, atol=1e-7)
        r0 += L


@pytest.mark.parametrize("int_attention", [False, True])
def test_calibrate_takes_each_scale_from_its_own_intermediate(int_attention):
    """OL.calibrate (P:72 'top 0.01%', R6; pipeline order P:121) on the
    zero-weight layer: s_qkv_in from h, s_attn from q|k|v = b^{QKV} (/127),
    s_o_in from OA = b^V, s_ffn1_in from LN1(b^A + h), s_ffn2_in from
    GELU(b^1) -- not from b^1 (pre-GELU) or from h1."""
    W = _zero_weight_layer()
    seqlens = [16, 16]
    M, d = sum(seqlens), W.hidden
    hc = synth.hidden_states(1, M, d, seed=1000000)
    OL.calibrate(hc, W, seqlens, int_attention=int_attention)
    tile = lambda v: np.tile(v, (M, 1))  # noqa: E731
    assert W.s_qkv_in == oracle.act_scale(hc, 7)
    bq = W.qkv.bias
    if int_attention:
        assert W.s_attn == oracle.act_scale(tile(bq), 127)
        # OA of the int8 core on identical keys is the exact mean of the v codes
        cv = oracle.quantize(bq[None, 2 * d:], W.s_attn, -127, 127)[0].astype(np.float32)
        oa = (cv * np.float32(W.s_attn)).astype(np.float32)
        assert np.isclose(W.s_o_in, oracle.act_scale(tile(oa), 7), rtol=1e-6)
    else:
        assert np.isclose(W.s_o_in, oracle.act_scale(tile(bq[2 * d:]), 7), rtol=1e-6)
    h1 = _ln_textbook(tile(W.o.bias).astype(np.float64) + hc, W.ln1_g, W.ln1_b)
    assert np.isclose(W.s_ffn1_in, oracle.act_scale(h1, 7), rtol=1e-6)
    g = tile(oracle.gelu_pinned(W.w1.bias))
    assert W.s_ffn2_in == oracle.act_scale(g, 7)
    assert W.s_ffn2_in != oracle.act_scale(tile(W.w1.bias), 7)
