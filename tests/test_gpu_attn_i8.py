"""GPU parity of the NEXT(2) integer attention core (mkq_attention_i8,
reading R19) against the oracle's attention_int8: bit-exact fp32 OA and
fused int4/int8 codes (the only non-integer step, the fp64 exp of the integer
score gap, is evaluated in the same fp64 operations on both sides)."""
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


def _codes(T, heads, seed, realistic):
    rng = np.random.default_rng(seed)
    if realistic:   # fp32 q|k|v ~ N(0,1) with outliers, Eq.1 to [-127,127] with a p99.99 scale
        x = synth.activations(T, 3 * 64 * heads, seed=seed)
        s = np.float32(oracle.abs_quantile(x, 0.9999)) / np.float32(127)
        return oracle.quantize(x, s, -127, 127), np.float32(s)
    return rng.integers(-127, 128, (T, 3 * 64 * heads)).astype(np.int8), np.float32(0.013)


@pytest.mark.parametrize("seqlens,heads", [([1, 17, 100, 5], 2), ([128], 12), ([33, 64, 2, 128, 31], 4),
                                           ([27] * 16, 12)])
@pytest.mark.parametrize("realistic", [False, True])
def test_attention_i8_bitexact(seqlens, heads, realistic):
    T = sum(seqlens)
    codes, s = _codes(T, heads, T + heads, realistic)
    cu = dev(np.concatenate([[0], np.cumsum(seqlens)]).astype(np.int32))
    ref = OL.attention_int8(codes, seqlens, heads, s)
    got = host(M.mkq_attention_i8(dev(codes), heads, len(seqlens), max(seqlens), s, cu, mode=M.OUT_F32))
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), np.abs(got - ref).max()
    for mode, lo, hi, so in ((M.OUT_I4, -8, 7, np.float32(0.05)), (M.OUT_I8, -128, 127, np.float32(0.004))):
        q = host(M.mkq_attention_i8(dev(codes), heads, len(seqlens), max(seqlens), s, cu, mode=mode, s_out=so,
                                    qmin=lo, qmax=hi))
        rq = oracle.quantize(ref, so, lo, hi)
        assert np.array_equal(q, oracle.pack_int4(rq)) if mode == M.OUT_I4 else np.array_equal(q.view(np.int8), rq)


def test_attention_i8_uniform_batch_and_errors():
    B, S, heads = 3, 64, 2
    codes, s = _codes(B * S, heads, 7, True)
    ref = OL.attention_int8(codes, [S] * B, heads, s)
    got = host(M.mkq_attention_i8(dev(codes), heads, B, S, s, None))
    assert np.array_equal(got, ref)
    from paper_2203_13483_b200._lib import MkqError
    with pytest.raises(MkqError):   # sequences longer than 128 are the fp16 kernels' job
        M.mkq_attention_i8(dev(np.zeros((130, 384), np.int8)), 2, 1, 130, s, None)


@pytest.mark.parametrize("s", [1e-3, 4e-3])
def test_attention_i8_small_scale_ragged_keys(s):
    """Small s_attn (c = s^2/8 tiny, so even the largest score gaps give
    p > 0) with L % 4 != 0: the padded key slots of the last 4-key group must
    contribute nothing (masked by index)."""
    seqlens, heads = [1, 5, 30, 127, 66, 3], 2
    T = sum(seqlens)
    codes, _ = _codes(T, heads, 99, False)
    s = np.float32(s)
    cu = dev(np.concatenate([[0], np.cumsum(seqlens)]).astype(np.int32))
    ref = OL.attention_int8(codes, seqlens, heads, s)
    got = host(M.mkq_attention_i8(dev(codes), heads, len(seqlens), max(seqlens), s, cu, mode=M.OUT_F32))
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), np.abs(got - ref).max()
