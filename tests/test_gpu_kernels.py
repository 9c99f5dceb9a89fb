"""GPU parity of every CUDA entry point against the CPU oracle, through the
C ABI (paper_2203_13483_b200.mkq -> libmkq.so).  Bit-exact on codes, int32
accumulators, fp32/fp16/bf16 epilogue outputs (the epilogue pins its fp32
op order, R4/R7/R11); tolerance only for the fp32 glue (attention,
LayerNorm) whose fused quantize is still checked bit-exactly against the
oracle applied to the GPU's own fp32 values (stage-wise replay)."""
import numpy as np
import pytest
import torch

import oracle
from oracle import layer as OL
import synth

pytestmark = pytest.mark.gpu

from paper_2203_13483_b200 import mkq as M  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    if t.dtype == torch.bfloat16:
        t = t.view(torch.int16)
    return t.cpu().numpy()


# ------------------------------------------------------------------ a1 quantize
@pytest.mark.parametrize("rows,cols", [(1, 32), (7, 96), (128, 768), (1000, 1024), (3, 6), (5, 1030)])
@pytest.mark.parametrize("bits", [4, 8])
def test_quantize_pack_parity(rows, cols, bits):
    x = synth.activations(rows, cols, seed=rows * 7 + cols)
    lo, hi = (-8, 7) if bits == 4 else (-128, 127)
    s = np.float32(0.5558) if bits == 4 else np.float32(0.0306)
    q = M.mkq_quantize_pack(dev(x), dev(np.array([s], np.float32)), bits, lo, hi)
    ref = oracle.quantize(x, s, lo, hi)
    if bits == 4:
        assert np.array_equal(host(q), oracle.pack_int4(ref))
    else:
        assert np.array_equal(host(q).view(np.int8), ref)


def test_quantize_per_row_weights_and_absmax():
    w = synth.weight(768, 1024, seed=3)
    s_gpu = M.mkq_absmax_scale(dev(w), 7.0, per_row=True)
    s_ref = oracle.absmax_scale(w, 7)
    assert np.array_equal(host(s_gpu), s_ref)
    q = M.mkq_quantize_pack(dev(w), s_gpu, 4, -7, 7, per_row=True)
    assert np.array_equal(host(q), oracle.pack_int4(oracle.quantize(w, s_ref, -7, 7, per_row=True)))
    st = M.mkq_absmax_scale(dev(w), 127.0, per_row=False)
    assert np.array_equal(host(st), oracle.absmax_scale(w, 127, per_row=False))


def test_quantize_ties_half_even():
    x = ((np.arange(-20, 20, dtype=np.float32) + np.float32(0.5)) * np.float32(0.25))[None, :].repeat(2, 0)
    q = M.mkq_quantize_pack(dev(x), dev(np.float32([0.25])), 8, -128, 127)
    assert np.array_equal(host(q).view(np.int8), oracle.quantize(x, np.float32(0.25), -128, 127))


# ------------------------------------------------------------------ a2-a7 GEMM
def _codes(rng, M_, N_, K_, bits):
    if bits == 4:
        A = rng.integers(-8, 8, (M_, K_)).astype(np.int8)
        W = rng.integers(-7, 8, (N_, K_)).astype(np.int8)
    else:
        A = rng.integers(-128, 128, (M_, K_)).astype(np.int8)
        W = rng.integers(-127, 128, (N_, K_)).astype(np.int8)
    return A, W


def _run(bits, A, W, s_a, s_w, b, **kw):
    K_ = A.shape[1]
    if bits == 4:
        return M.mkq_gemm_w4a4(dev(oracle.pack_int4(A)), dev(oracle.pack_int4(W)), s_a, dev(s_w),
                               None if b is None else dev(b), K=K_, **kw)
    return M.mkq_gemm_w8a8(dev(A), dev(W), s_a, dev(s_w), None if b is None else dev(b), K=K_, **kw)


SHAPES = [(1, 32, 32), (7, 64, 96), (128, 768, 768), (129, 256, 160), (300, 512, 1024), (257, 288, 64),
          (1000, 3072, 768)]


@pytest.fixture(params=[-1, 0, 1, 2], ids=["plan-auto", "plan-large", "plan-small", "plan-mma"])
def small_mode(request):
    """GEMM tile plan: heuristic, never / always the small-M split-K plan."""
    from paper_2203_13483_b200._lib import lib
    lib().mkq_set_small_m_mode(request.param)
    yield request.param
    lib().mkq_set_small_m_mode(-1)


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("Mm,N,K", SHAPES)
def test_gemm_raw_i32_bitexact(bits, Mm, N, K, small_mode):
    rng = np.random.default_rng(Mm * 31 + N + K)
    A, W = _codes(rng, Mm, N, K, bits)
    out = _run(bits, A, W, 1.0, np.ones(N, np.float32), None, mode=M.OUT_I32)
    assert np.array_equal(host(out), oracle.gemm_i32(A, W))


# Table-2 sized GEMMs (BERT-base, 440 / 2298 valid tokens) through the small-M
# split-K plan, every epilogue mode, repeated calls (self-resetting counters)
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("Mm,N,K", [(440, 768, 3072), (440, 2304, 768), (440, 3072, 768), (440, 768, 768),
                                     (1, 768, 3072), (130, 64, 4096), (2298, 768, 768)])
@pytest.mark.parametrize("plan", [1, 2])
def test_gemm_small_m_split_k(bits, Mm, N, K, plan):
    from paper_2203_13483_b200._lib import lib
    lib().mkq_set_small_m_mode(plan)
    try:
        rng = np.random.default_rng(Mm + N + K + bits)
        A, W = _codes(rng, Mm, N, K, bits)
        ref = oracle.gemm_i32(A, W)
        for _ in range(3):
            assert np.array_equal(host(_run(bits, A, W, 1.0, np.ones(N, np.float32), None, mode=M.OUT_I32)), ref)
        lo, hi = (-8, 7) if bits == 4 else (-128, 127)
        s_a = np.float32(0.31 if bits == 4 else 0.0306)
        s_w = rng.uniform(1e-3, 5e-3, N).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
        out = host(_run(bits, A, W, s_a, s_w, b, mode=M.OUT_F32))
        assert np.array_equal(out.view(np.uint32), oracle.linear(A, W, s_a, s_w, b).view(np.uint32))
        s_out = np.float32(0.05 if bits == 4 else 0.004)
        mode = M.OUT_I4 if bits == 4 else M.OUT_I8
        r = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_I4 if bits == 4 else oracle.OUT_I8, gelu=True,
                          s_out=s_out, qmin_out=lo, qmax_out=hi)
        for table in (True, False):   # exact requant table / direct GELU + division
            out = host(_run(bits, A, W, s_a, s_w, b, mode=mode, gelu=True, s_out=s_out, qmin=lo, qmax=hi,
                            requant_table=table))
            assert np.array_equal(out, oracle.pack_int4(r)) if bits == 4 else np.array_equal(out.view(np.int8), r)
    finally:
        lib().mkq_set_small_m_mode(-1)


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("mode", [M.OUT_F32, M.OUT_F16, M.OUT_BF16])
@pytest.mark.parametrize("gelu", [False, True])
def test_gemm_float_epilogues_bitexact(bits, mode, gelu, small_mode):
    rng = np.random.default_rng(17 + mode)
    Mm, N, K = 300, 768, 1024
    A, W = _codes(rng, Mm, N, K, bits)
    s_a = np.float32(0.5558 if bits == 4 else 0.0306)
    s_w = rng.uniform(1e-3, 1e-2, N).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    out = host(_run(bits, A, W, s_a, s_w, b, mode=mode, gelu=gelu))
    omode = {M.OUT_F32: oracle.OUT_F32, M.OUT_F16: oracle.OUT_F16, M.OUT_BF16: oracle.OUT_BF16}[mode]
    ref = oracle.linear(A, W, s_a, s_w, b, mode=omode, gelu=gelu)
    if mode == M.OUT_F32:
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
    else:
        assert np.array_equal(out.view(np.uint16), ref.view(np.uint16))


# int4 small M with more 128 x 64 tiles than SMs but 128 x 128 tiles in one
# wave (Table-2 QKV at 537-681 tokens): the 128 x 128 A-in-TMEM plan, every
# plain output mode (GELU included) and the raw accumulators
@pytest.mark.parametrize("Mm,N,K", [(681, 2304, 768), (900, 1280, 1024), (537, 2304, 96)])
@pytest.mark.parametrize("mode", [M.OUT_F32, M.OUT_F16, M.OUT_BF16, M.OUT_I32])
def test_gemm_small_m_wide_tiles(Mm, N, K, mode):
    rng = np.random.default_rng(Mm + N + K + mode)
    A, W = _codes(rng, Mm, N, K, 4)
    s_a = np.float32(0.5558)
    s_w = rng.uniform(1e-3, 1e-2, N).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    gelu = mode == M.OUT_F32
    out = host(_run(4, A, W, s_a, s_w, b, mode=mode, gelu=gelu))
    if mode == M.OUT_I32:
        assert np.array_equal(out, oracle.gemm_i32(A, W))
        return
    omode = {M.OUT_F32: oracle.OUT_F32, M.OUT_F16: oracle.OUT_F16, M.OUT_BF16: oracle.OUT_BF16}[mode]
    ref = oracle.linear(A, W, s_a, s_w, b, mode=omode, gelu=gelu)
    if mode == M.OUT_F32:
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
    else:
        assert np.array_equal(out.view(np.uint16), ref.view(np.uint16))


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("Mm,N,K", [(1, 32, 64), (128, 3072, 768), (257, 4096, 1024)])
def test_gemm_requant_gelu_bitexact(bits, Mm, N, K, small_mode):
    rng = np.random.default_rng(5 + Mm)
    A, W = _codes(rng, Mm, N, K, bits)
    lo, hi = (-8, 7) if bits == 4 else (-128, 127)
    s_a = np.float32(0.31)
    s_w = rng.uniform(1e-3, 5e-3, N).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    s_out = np.float32(0.05 if bits == 4 else 0.004)
    mode = M.OUT_I4 if bits == 4 else M.OUT_I8
    for gelu in (False, True):
        out = host(_run(bits, A, W, s_a, s_w, b, mode=mode, gelu=gelu, s_out=s_out, qmin=lo, qmax=hi))
        ref = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_I4 if bits == 4 else oracle.OUT_I8, gelu=gelu,
                            s_out=s_out, qmin_out=lo, qmax_out=hi)
        if bits == 4:
            assert np.array_equal(out, oracle.pack_int4(ref))
        else:
            assert np.array_equal(out.view(np.int8), ref)


def test_gemm_worst_case_magnitudes():
    K = 4096
    for a, w, exp in [(-8, -7, 229376), (-8, 7, -229376), (7, 7, 200704)]:
        A = np.full((130, K), a, np.int8)
        W = np.full((64, K), w, np.int8)
        out = host(_run(4, A, W, 1.0, np.ones(64, np.float32), None, mode=M.OUT_I32))
        assert np.all(out == exp)
    A = np.full((130, K), -128, np.int8)
    W = np.full((64, K), -127, np.int8)
    out = host(_run(8, A, W, 1.0, np.ones(64, np.float32), None, mode=M.OUT_I32))
    assert np.all(out == 66584576)


@pytest.mark.parametrize("small", [0, 1, 2])
def test_gemm_max_k_extremes(small):
    """K = MKQ_MAX_K = 131040 (the exactness limit of include/mkq.h): the
    int4 accumulator holds 256 * sum = 256 * 64 * 131040 = 2147000320 < 2^31
    for A = W = -8 (any nibble is a valid int4 code), through both GEMM plans;
    int8 at the same K with |a w| = 128 * 127."""
    from paper_2203_13483_b200._lib import lib
    lib().mkq_set_small_m_mode(small)
    try:
        K = 131040
        for a, w in ((-8, -8), (7, -8)):
            A = np.full((3, K), a, np.int8)
            W = np.full((32, K), w, np.int8)
            out = host(_run(4, A, W, 1.0, np.ones(32, np.float32), None, mode=M.OUT_I32))
            assert np.all(out == a * w * K)
        A = np.full((3, K), -128, np.int8)
        W = np.full((32, K), 127, np.int8)
        out = host(_run(8, A, W, 1.0, np.ones(32, np.float32), None, mode=M.OUT_I32))
        assert np.all(out == -128 * 127 * K)
        rng = np.random.default_rng(1)
        A, W = _codes(rng, 5, 64, K, 4)
        assert np.array_equal(host(_run(4, A, W, 1.0, np.ones(64, np.float32), None, mode=M.OUT_I32)),
                              oracle.gemm_i32(A, W))
    finally:
        lib().mkq_set_small_m_mode(-1)


def test_degenerate_sizes():
    """M = 0 is a no-op; the smallest legal GEMM (1 x 32 x 32); one-token
    sequences in attention; a single LayerNorm row."""
    rng = np.random.default_rng(2)
    A, W = _codes(rng, 1, 32, 32, 4)
    assert np.array_equal(host(_run(4, A, W, 1.0, np.ones(32, np.float32), None, mode=M.OUT_I32)),
                          oracle.gemm_i32(A, W))
    z = torch.empty((0, 16), dtype=torch.uint8, device=DEV)
    o = M.mkq_gemm_w4a4(z, dev(oracle.pack_int4(W)), 1.0, dev(np.ones(32, np.float32)), None,
                        mode=M.OUT_I32, out=torch.empty((0, 32), dtype=torch.int32, device=DEV), K=32)
    assert o.shape == (0, 32)
    # attention over three 1-token sequences: softmax of one score is 1, OA = v
    qkv = (rng.standard_normal((3, 3 * 128)) * 0.5).astype(np.float16)
    cu = dev(np.array([0, 1, 2, 3], np.int32))
    oa = host(M.mkq_attention(dev(qkv), 2, 3, 1, cu, mode=M.OUT_F32))
    assert np.allclose(oa, qkv[:, 256:].astype(np.float32), rtol=1e-3, atol=1e-3)
    x = synth.activations(1, 768, seed=4)
    y = host(M.mkq_residual_layernorm(dev(x), None, dev(np.ones(768, np.float32)),
                                      dev(np.zeros(768, np.float32)), 1e-12))
    ref = OL.layernorm(x.astype(np.float64), np.ones(768, np.float32), np.zeros(768, np.float32))
    assert np.abs(y - ref).max() < 2e-5


def test_gemm_zero_rows_and_strided():
    rng = np.random.default_rng(9)
    A, W = _codes(rng, 100, 256, 512, 4)
    A[13] = 0
    Ap = oracle.pack_int4(A)
    big = np.zeros((100, 512), np.uint8)          # lda = 512 bytes > K/2
    big[:, :256] = Ap
    a_t = dev(big)[:, :256]
    out = torch.zeros((100, 300), dtype=torch.int32, device=DEV)[:, :256]   # ldo > N*4
    M.mkq_gemm_w4a4(a_t, dev(oracle.pack_int4(W)), 1.0, dev(np.ones(256, np.float32)), None,
                    mode=M.OUT_I32, out=out, K=512)
    ref = oracle.gemm_i32(A, W)
    assert np.array_equal(host(out), ref)
    assert np.all(host(out)[13] == 0)


def test_w8a8_equals_w4a4_when_codes_fit():
    rng = np.random.default_rng(10)
    A, W = _codes(rng, 200, 512, 768, 4)
    o4 = host(_run(4, A, W, 1.0, np.ones(512, np.float32), None, mode=M.OUT_I32))
    o8 = host(_run(8, A, W, 1.0, np.ones(512, np.float32), None, mode=M.OUT_I32))
    assert np.array_equal(o4, o8)


@pytest.mark.parametrize("N,K", [(4096, 1024), (1024, 4096), (3072, 1024)])
def test_gemm_full_size_sampled_rows(N, K):
    """BASELINE configs[3] shapes at full M (131072 rows, the bench launch
    configuration): GPU computes everything, the oracle a sample of rows."""
    Mm = 131072
    rng = np.random.default_rng(N + K)
    A = rng.integers(-8, 8, (Mm, K)).astype(np.int8)
    W = rng.integers(-7, 8, (N, K)).astype(np.int8)
    s_w = rng.uniform(1e-3, 5e-3, N).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    Ap = dev(oracle.pack_int4(A))
    Wp = dev(oracle.pack_int4(W))
    out = host(M.mkq_gemm_w4a4(Ap, Wp, 0.31, dev(s_w), dev(b), mode=M.OUT_F32, K=K))
    rows = np.sort(rng.choice(Mm, 48, replace=False))
    rows[-1] = Mm - 1
    ref = oracle.linear(A[rows], W, np.float32(0.31), s_w, b, mode=oracle.OUT_F32)
    assert np.array_equal(out[rows].view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------------------ a8 glue
def _qkv_fp16(T, hidden, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((T, 3 * hidden)).astype(np.float32) * np.float32(0.8)).astype(np.float16)


@pytest.mark.parametrize("seqlens,heads", [([128], 12), ([64, 64], 2), ([1, 17, 130, 5], 4), ([512, 512], 16)])
def test_attention_vs_oracle(seqlens, heads):
    T = sum(seqlens)
    hidden = heads * 64
    qkv = _qkv_fp16(T, hidden, seed=T)
    cu = np.concatenate([[0], np.cumsum(seqlens)]).astype(np.int32)
    uniform = len(set(seqlens)) == 1
    out = host(M.mkq_attention(dev(qkv), heads, len(seqlens), max(seqlens),
                               None if uniform else dev(cu), mode=M.OUT_F32))
    ref = OL.attention(qkv.astype(np.float64), seqlens, heads)
    err = np.abs(out - ref)
    assert err.max() < 2e-3 * max(1.0, np.abs(ref).max()), err.max()
    # fused quantize == oracle quantize of the GPU's own fp32 OA (bit-exact)
    s = np.float32(0.05)
    q = host(M.mkq_attention(dev(qkv), heads, len(seqlens), max(seqlens), None if uniform else dev(cu),
                             mode=M.OUT_I4, s_out=s))
    assert np.array_equal(q, oracle.pack_int4(oracle.quantize(out, s, -8, 7)))


@pytest.mark.parametrize("rows,cols", [(5, 768), (300, 1024), (17, 4096)])
def test_residual_layernorm(rows, cols):
    rng = np.random.default_rng(rows + cols)
    x = rng.standard_normal((rows, cols)).astype(np.float32) * 3
    r = rng.standard_normal((rows, cols)).astype(np.float32)
    g, b = synth.ln_params(cols, 3)
    y, q = M.mkq_residual_layernorm(dev(x), dev(r), dev(g), dev(b), 1e-12, bits=4, s_q=0.5558)
    y = host(y)
    ref = OL.layernorm(x.astype(np.float64) + r, g, b)
    assert np.abs(y - ref).max() < 2e-5 * max(1.0, np.abs(ref).max())
    assert np.array_equal(host(q), oracle.pack_int4(oracle.quantize(y, np.float32(0.5558), -8, 7)))


# ------------------------------------------------------------------ errors on device
def test_device_errors_surface():
    with pytest.raises(M.__dict__.get("MkqError", RuntimeError)):
        M.mkq_gemm_w4a4(torch.zeros((4, 16), dtype=torch.uint8, device=DEV),
                        torch.zeros((33, 16), dtype=torch.uint8, device=DEV), 1.0,
                        torch.ones(33, device=DEV))


# ------------------------------------------------------------------ requant table (a5/a6 fused)
@pytest.mark.parametrize("gelu,s_out,bits", [(True, 0.05, 4), (True, 0.6, 4), (True, 3.0, 4), (False, 0.3, 4),
                                             (True, 0.004, 8), (True, 0.04, 8), (False, 0.01, 8)])
def test_requant_table_bitexact(gelu, s_out, bits):
    lo, hi = (-8, 7) if bits == 4 else (-128, 127)
    tab = M.mkq_requant_table(gelu, s_out, lo, hi, DEV, cache=False)
    torch.cuda.synchronize()
    assert int(tab[28:32].view(torch.int32).item()) == 1, "table self-verification failed"
    if bits == 4 and s_out >= 0.05:   # the compact int4 table (FFN1 fast path) must be usable too
        assert int(tab[TAB4 + 8:TAB4 + 12].view(torch.int32).item()) == 1, "compact table not valid"
    rng = np.random.default_rng(int(s_out * 1000) + bits)
    Mm, N, K = 1000, 1024, 1024
    A, W = _codes(rng, Mm, N, K, bits)
    s_a = np.float32(0.31 if bits == 4 else 0.02)
    s_w = rng.uniform(1e-3, 5e-3, N).astype(np.float32) if bits == 4 else rng.uniform(1e-4, 3e-4, N).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    mode = M.OUT_I4 if bits == 4 else M.OUT_I8
    with_t = host(_run(bits, A, W, s_a, s_w, b, mode=mode, gelu=gelu, s_out=s_out, qmin=lo, qmax=hi,
                       requant_table=tab))
    without = host(_run(bits, A, W, s_a, s_w, b, mode=mode, gelu=gelu, s_out=s_out, qmin=lo, qmax=hi,
                        requant_table=None))
    assert np.array_equal(with_t, without)
    ref = oracle.linear(A, W, s_a, s_w, b, mode=oracle.OUT_I4 if bits == 4 else oracle.OUT_I8, gelu=gelu,
                        s_out=np.float32(s_out), qmin_out=lo, qmax_out=hi)
    assert np.array_equal(with_t if bits == 4 else with_t.view(np.int8), oracle.pack_int4(ref) if bits == 4 else ref)


TAB4 = 64 + 1024 * 8   # byte offset of the compact int4 table header (requant.cuh kOff4)


@pytest.mark.parametrize("s_out", [0.36, 0.05])
def test_requant_table4_threshold_neighbourhoods(s_out):
    """The compact table word keeps the threshold only to a 256-float run: drive y
    through +-600 ulps around every threshold word (acc = 0, so y = bias
    exactly) and through the non-folded (tiny scale) epilogue; every code
    must equal the oracle's direct evaluation."""
    tab = M.mkq_requant_table(True, s_out, -8, 7, DEV, cache=False)
    torch.cuda.synchronize()
    t = tab.cpu().numpy()
    assert t[TAB4 + 8:TAB4 + 12].view(np.int32)[0] == 1
    words = t[TAB4 + 64:TAB4 + 64 + 256 * 4].view(np.uint32)
    thr = words[(words & 0x7F800000) != 0x7F800000]
    assert thr.size >= 5
    ys = np.unique(np.concatenate([(w.astype(np.int64) + np.arange(-600, 601)) for w in thr]).astype(np.uint32))
    ys = ys.view(np.float32)
    N = (ys.size + 255) // 256 * 256
    b = np.resize(ys, N).astype(np.float32)
    rng = np.random.default_rng(11)
    K = 256
    A = np.zeros((256, K), np.int8)
    W = rng.integers(-7, 8, (N, K)).astype(np.int8)
    s_w = np.full(N, 2e-3, np.float32)
    s_w[N // 2: N // 2 + 256] = 1e-37   # one tile with an unfoldable (tiny) scale
    out = host(_run(4, A, W, np.float32(0.3), s_w, b, mode=M.OUT_I4, gelu=True, s_out=s_out, requant_table=tab))
    ref = oracle.linear(A, W, np.float32(0.3), s_w, b, mode=oracle.OUT_I4, gelu=True, s_out=np.float32(s_out))
    assert np.array_equal(out, oracle.pack_int4(ref))


def test_requant_table_mismatched_params_ignored():
    """A table built for other (gelu, s_out, range) must not be used."""
    tab = M.mkq_requant_table(True, 0.5, -8, 7, DEV, cache=False)
    rng = np.random.default_rng(3)
    A, W = _codes(rng, 512, 512, 512, 4)
    s_w = rng.uniform(1e-3, 5e-3, 512).astype(np.float32)
    out = host(_run(4, A, W, 0.3, s_w, None, mode=M.OUT_I4, gelu=True, s_out=0.07, requant_table=tab))
    ref = oracle.linear(A, W, np.float32(0.3), s_w, None, mode=oracle.OUT_I4, gelu=True, s_out=np.float32(0.07))
    assert np.array_equal(out, oracle.pack_int4(ref))
