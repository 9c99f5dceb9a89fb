"""GPU parity of the QAT-side kernels
and the GPU calibration statistic (NEXT(4)) against the CPU oracle,
through the C ABI.

Bar: fake-quant values, STE input gradients and the calibration scale are
bit-exact.  The two fp64 scale-gradient sums differ from the oracle's
term-by-term sums only by summation order; the test bound is the standard
one for recursive/pairwise fp64 summation, 4 n u sum|terms| with u = 2^-53
(DESIGN.md §4), applied to the sum of absolute terms of each gradient."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

from paper_2203_13483_b200 import mkq as M  # noqa: E402

DEV = "cuda:0"
U = 2.0 ** -53


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _grad_bounds(x, s, lo, hi):
    """Sum of |terms| of each scale gradient (for the summation-order bound)."""
    x64 = x.astype(np.float64)
    q = oracle.quantize(x.reshape(1, -1), s, lo, hi).ravel().astype(np.float64) if x.size else np.zeros(0)
    ste_abs = np.sum(np.abs(x64) / np.float64(s)) + np.sum(np.abs(q))
    mse_abs = 2 * (np.float64(s) * np.sum(q * q) + np.sum(np.abs(x64 * q)))
    return ste_abs, mse_abs


def _check(x, s, lo, hi, gy, offset=0):
    n = x.size
    if offset:
        # misaligned views (4-byte offset) take the scalar path
        xb = dev(np.concatenate([np.zeros(offset, np.float32), x]))
        gb = dev(np.concatenate([np.zeros(offset, np.float32), gy]))
        xd, gd = xb[offset:], gb[offset:]
    else:
        xd, gd = dev(x), dev(gy)
    y, gx, gs = M.mkq_fake_quant(xd, dev(np.array([s], np.float32)), lo, hi, grad_y=gd)
    assert np.array_equal(host(y).view(np.uint32), oracle.fake_quant(x, s, lo, hi).view(np.uint32))
    assert np.array_equal(host(gx).view(np.uint32), oracle.ste_grad_x(x, gy, s, lo, hi).view(np.uint32))
    g = host(gs)
    ste_abs, mse_abs = _grad_bounds(x, s, lo, hi)
    tol = 4 * max(n, 1) * U
    assert abs(g[0] - oracle.scale_grad_ste(x, s, lo, hi)) <= tol * ste_abs + 1e-300
    assert abs(g[1] - oracle.scale_grad_mse(x, s, lo, hi)) <= tol * mse_abs + 1e-300
    return g


@pytest.mark.parametrize("n", [0, 1, 5, 1023, 4099, 1_000_003])
@pytest.mark.parametrize("bits", [4, 8])
def test_fake_quant_parity(n, bits):
    x = synth.activations(1, n, seed=n + bits).ravel() if n else np.zeros(0, np.float32)
    gy = np.random.default_rng(n).standard_normal(n).astype(np.float32)
    lo, hi, s = (-8, 7, np.float32(0.5558)) if bits == 4 else (-128, 127, np.float32(0.0306))
    g = _check(x, s, lo, hi, gy)
    if n == 0:
        assert g.tolist() == [0.0, 0.0]


def test_fake_quant_misaligned_and_ties():
    # exact ties (n + 1/2) s with s a power of two, both signs, around the clamp bounds
    s = np.float32(0.25)
    x = ((np.arange(-12, 12, dtype=np.float32) + np.float32(0.5)) * s)
    x = np.concatenate([x, synth.activations(1, 3001, seed=5).ravel()])
    gy = np.random.default_rng(1).standard_normal(x.size).astype(np.float32)
    _check(x, s, -8, 7, gy, offset=1)
    _check(x, s, -8, 7, gy, offset=0)


def test_fake_quant_paper_example_and_clipping():
    """P:145-151 / P:187 on the GPU, plus the hand-worked clipped case of
    tests/test_oracle.py (STE -0.8, MSE -24.2)."""
    for xs, ste, mse in (([0.2, 0.9], -0.1, 0.2), ([0.2, 0.9, -0.3, 7.6, -9.0], -0.8, -24.2)):
        x = np.array(xs, np.float32)
        _, _, gs = M.mkq_fake_quant(dev(x), dev(np.array([1.0], np.float32)), -8, 7)
        g = host(gs)
        assert g[0] == pytest.approx(ste, abs=1e-6) and g[1] == pytest.approx(mse, abs=1e-5)


def test_fake_quant_deterministic_and_large():
    n = (1 << 24) + 7
    x = synth.activations(1, n, seed=77).ravel()
    gy = np.ones(n, np.float32)
    g1 = _check(x, np.float32(0.5558), -8, 7, gy)
    _, _, gs = M.mkq_fake_quant(dev(x), dev(np.array([0.5558], np.float32)), -8, 7)
    assert np.array_equal(host(gs), g1)   # same grid, fixed fold order


def test_fake_quant_errors():
    x = dev(np.ones(8, np.float32))
    sc = dev(np.array([1.0], np.float32))
    from paper_2203_13483_b200._lib import MkqError
    with pytest.raises(MkqError):
        M.mkq_fake_quant(x, sc, 7, 7)


# ------------------------------------------------------------------ calibration
@pytest.mark.parametrize("n", [1, 2, 4, 100, 4097, 1_000_003])
@pytest.mark.parametrize("p", [0.0, 0.5, 0.9999, 1.0])
def test_act_scale_parity(n, p):
    x = synth.activations(1, n, seed=n).ravel()
    got = host(M.mkq_act_scale(dev(x), 7.0, p))[0]
    ref = np.float32(oracle.abs_quantile(x, p)) / np.float32(7)
    assert got.view(np.uint32) == np.float32(ref).view(np.uint32), (got, ref)


def test_act_scale_duplicates_zeros_misaligned():
    rng = np.random.default_rng(4)
    cases = [np.zeros(1000, np.float32), np.full(777, -3.5, np.float32),
             rng.integers(-3, 4, 100_001).astype(np.float32),           # heavy ties in the order statistics
             (rng.standard_cauchy(200_000)).astype(np.float32),          # heavy tail
             np.concatenate([np.zeros(5000, np.float32), np.float32(1e-40) * np.ones(3, np.float32)])]  # subnormals
    for x in cases:
        for p in (0.9999, 0.37, 1.0):
            ref = np.float32(oracle.abs_quantile(x, p)) / np.float32(7)
            got = host(M.mkq_act_scale(dev(x), 7.0, p))[0]
            assert got.view(np.uint32) == np.float32(ref).view(np.uint32), (x[:4], p, got, ref)
            xb = dev(np.concatenate([np.zeros(1, np.float32), x]))[1:]      # 4-byte offset: scalar path
            got = host(M.mkq_act_scale(xb, 7.0, p))[0]
            assert got.view(np.uint32) == np.float32(ref).view(np.uint32)


def test_act_scale_full_size_calibration_tensor():
    """A BASELINE configs[3]-shaped slab (16 sequences of 512 x 1024 = 8.4 M
    values, N(0,1) + outliers): bit-exact against the oracle's sort."""
    x = synth.activations(16 * 512, 1024, seed=9).ravel()
    got = host(M.mkq_act_scale(dev(x), 7.0, 0.9999))[0]
    ref = np.float32(oracle.abs_quantile(x, 0.9999)) / np.float32(7)
    assert got.view(np.uint32) == np.float32(ref).view(np.uint32)
