"""NEXT(4) fused glue: mkq_gemm_residual_ln (W4A4 GEMM + residual + post-LN
[+ Eq.1 codes], one kernel, row statistics exchanged between the CTA pairs
of a row group) against the CPU oracle.  The dequant is the plain epilogue's
exact fp32 sequence (R4), so the oracle's r = fl32(linear + res) is the GPU's
LN input bit for bit; LN itself is a tolerance stage (fp32 vs the fp64
oracle, the residual_ln bar 2e-5 max(1,|ref|)); the codes are bit-exact
against the oracle quantizer applied to the GPU's own LN output."""
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
    return t.cpu().numpy()


def _case(Mr, N, K, seed, tiny_scale=False):
    rng = np.random.default_rng(seed)
    A = rng.integers(-8, 8, (Mr, K)).astype(np.int8)
    W = rng.integers(-7, 8, (N, K)).astype(np.int8)
    s_a = np.float32(0.05)
    s_w = rng.uniform(1e-3, 3e-3, N).astype(np.float32)
    if tiny_scale:
        s_w[N // 3] = np.float32(1e-37)   # a column scale too small for the 2^-8 fold
    b = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    res = synth.hidden_states(1, Mr, N, seed=seed + 1).reshape(Mr, N)
    g = (1 + 0.02 * rng.standard_normal(N)).astype(np.float32)
    beta = (0.02 * rng.standard_normal(N)).astype(np.float32)
    return A, W, s_a, s_w, b, res, g, beta


@pytest.mark.parametrize("Mr,N,K", [(256, 256, 256), (300, 1024, 1024), (1, 768, 512), (4096, 1024, 1024),
                                    (1000, 768, 3072), (2311, 512, 4096), (440, 768, 768), (440, 768, 3072),
                                    (130, 512, 96)])
@pytest.mark.parametrize("q_bits", [0, 4, 8])
@pytest.mark.parametrize("plan", [-1, 0], ids=["plan-auto", "plan-2cta"])
def test_gemm_residual_ln_parity(Mr, N, K, q_bits, plan):
    """plan-auto: M <= 128 x (co-resident N/64-CTA clusters) takes the small-M
    N-cluster kernel (row statistics over DSMEM), larger M the 2-CTA kernel;
    plan-2cta forces the 2-CTA kernel (mkq_set_small_m_mode(0))."""
    from paper_2203_13483_b200._lib import lib
    lib().mkq_set_small_m_mode(plan)
    try:
        _parity(Mr, N, K, q_bits)
    finally:
        lib().mkq_set_small_m_mode(-1)


def _parity(Mr, N, K, q_bits):
    A, W, s_a, s_w, b, res, g, beta = _case(Mr, N, K, seed=Mr + N + K + q_bits)
    a_d = dev(oracle.pack_int4(A))
    w_d = dev(oracle.pack_int4(W))
    lo, hi = (-8, 7) if q_bits == 4 else (-128, 127)
    s_q = np.float32(0.6 if q_bits == 4 else 0.03)
    out = M.mkq_gemm_residual_ln(a_d, w_d, float(s_a), dev(s_w), dev(b), dev(res), dev(g), dev(beta), 1e-12, K=K,
                                 q_bits=q_bits, s_q=float(s_q), qmin=lo, qmax=hi)
    y_d, q_d = out if q_bits else (out, None)
    y = host(y_d)
    lin = oracle.linear(A, W, s_a, s_w, b)                       # exact fp32 dequant (R4)
    r = (lin + res).astype(np.float32)                           # fl32 residual add (R9)
    ref = OL.layernorm(r, g, beta)
    assert np.abs(y - ref).max() < 2e-5 * max(1.0, np.abs(ref).max())
    if q_bits:
        codes = oracle.quantize(y, s_q, lo, hi)
        got = host(q_d)
        assert np.array_equal(got, oracle.pack_int4(codes)) if q_bits == 4 else np.array_equal(got.view(np.int8), codes)
    # agrees with the unfused GPU path (GEMM fp32 + residual_ln) within LN rounding
    o = M.mkq_gemm_w4a4(a_d, w_d, float(s_a), dev(s_w), dev(b), mode=M.OUT_F32, K=K)
    assert np.array_equal(host(o), lin)
    y2 = host(M.mkq_residual_layernorm(o, dev(res), dev(g), dev(beta), 1e-12))
    assert np.abs(y - y2).max() < 1e-5 * max(1.0, np.abs(ref).max())


def test_gemm_residual_ln_deterministic_and_unfolded_scale():
    """Fixed-order row statistics: two calls give identical bits; a tile with
    an unfoldable (tiny) column scale takes the shifted-accumulator dequant."""
    Mr, N, K = 1024, 1024, 1024
    A, W, s_a, s_w, b, res, g, beta = _case(Mr, N, K, seed=5, tiny_scale=True)
    args = (dev(oracle.pack_int4(A)), dev(oracle.pack_int4(W)), float(s_a), dev(s_w), dev(b), dev(res), dev(g),
            dev(beta), 1e-12)
    y1 = host(M.mkq_gemm_residual_ln(*args, K=K))
    y2 = host(M.mkq_gemm_residual_ln(*args, K=K))
    assert np.array_equal(y1, y2)
    ref = OL.layernorm((oracle.linear(A, W, s_a, s_w, b) + res).astype(np.float32), g, beta)
    assert np.abs(y1 - ref).max() < 2e-5 * max(1.0, np.abs(ref).max())


def test_gemm_residual_ln_validation():
    a = torch.zeros((256, 128), dtype=torch.uint8, device=DEV)
    w = torch.zeros((300, 128), dtype=torch.uint8, device=DEV)   # N not a multiple of 256
    f = torch.ones(300, device=DEV)
    from paper_2203_13483_b200._lib import MkqError
    with pytest.raises(MkqError):
        M.mkq_gemm_residual_ln(a, w, 1.0, f, None, torch.zeros((256, 300), device=DEV), f, f)
