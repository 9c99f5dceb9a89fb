"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; diagnostics).

    compute-sanitizer --tool memcheck python tools/sanitize_all.py [--part all|gemm|attn|glue|layer]

Covers: quantize / absmax, the 2-CTA W4A4 GEMM (every output mode, direct and
table requant, the compact-table FFN1 epilogue), the fused GEMM + residual +
LayerNorm kernel, the 1-CTA W8A8 GEMM, the small-M cluster split-K plan and
the mma.sync small-M kernel, both fp16 attention kernels and the integer one,
residual LayerNorm, fake-quant + gradients, the p99.99 calibration, the
requant-table builder, the block interleave, and two layers with the fused
cross-layer codes."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2203_13483_b200 import mkq as M, model  # noqa: E402
from paper_2203_13483_b200._lib import lib  # noqa: E402

dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)


def rnd_u8(r, c):
    return torch.randint(0, 256, (r, c), dtype=torch.uint8, device=dev, generator=g)


def part_gemm():
    sw = torch.rand(1024, device=dev, generator=g) * 1e-3 + 1e-4
    b = torch.rand(1024, device=dev, generator=g) * 0.1
    A, W = rnd_u8(300, 256), rnd_u8(512, 256)            # M ragged, K = 512
    for mode in (M.OUT_F32, M.OUT_F16, M.OUT_BF16, M.OUT_I4, M.OUT_I8, M.OUT_I32):
        i8 = mode == M.OUT_I8
        for tab in (True, False):
            M.mkq_gemm_w4a4(A, W, 0.3, sw[:512], b[:512], mode=mode, gelu=mode in (M.OUT_I4, M.OUT_I8), s_out=0.05,
                            qmin=-128 if i8 else -8, qmax=127 if i8 else 7, K=512, requant_table=tab)
    A8, W8 = rnd_u8(300, 512).view(torch.int8), rnd_u8(512, 512).view(torch.int8)
    M.mkq_gemm_w8a8(A8, W8, 0.3, sw[:512], b[:512], mode=M.OUT_F32, K=512)
    for mode_small in (1, 2):                            # small-M cluster split-K, mma.sync small-M
        lib().mkq_set_small_m_mode(mode_small)
        M.mkq_gemm_w4a4(rnd_u8(130, 256), W, 0.3, sw[:512], b[:512], mode=M.OUT_F32, K=512)
        M.mkq_gemm_w4a4(rnd_u8(130, 1536), rnd_u8(256, 1536), 0.3, sw[:256], b[:256], mode=M.OUT_I4, gelu=True,
                        s_out=0.05, K=3072)
        # small-M plan, unsplit: A in TMEM, TMA-stored epilogue (fp16 out, the QKV shape class)
        M.mkq_gemm_w4a4(rnd_u8(200, 384), rnd_u8(256, 384), 0.3, sw[:256], b[:256], mode=M.OUT_F16, K=768)
    lib().mkq_set_small_m_mode(-1)
    # Table-2 FFN1: GELU + int4 requant through the compact table on 256 x 128 CTA-pair tiles
    sw3 = torch.rand(3072, device=dev, generator=g) * 1e-3 + 1e-4
    b3 = torch.rand(3072, device=dev, generator=g) * 0.1
    M.mkq_gemm_w4a4(rnd_u8(440, 384), rnd_u8(3072, 384), 0.3, sw3, b3, mode=M.OUT_I4, gelu=True, s_out=0.05, K=768,
                    requant_table=True)
    # fused GEMM + residual + LN (+ codes), N = 768: the small-M N-cluster kernel (auto at
    # M = 300) and the 2-CTA kernel (three CTA pairs per row group; plan mode 0)
    res = torch.randn(300, 768, device=dev, generator=g)
    one, zero = torch.ones(768, device=dev), torch.zeros(768, device=dev)
    for plan in (-1, 0):
        lib().mkq_set_small_m_mode(plan)
        for qb in (0, 4, 8):
            M.mkq_gemm_residual_ln(rnd_u8(300, 256), rnd_u8(768, 256), 0.3, sw[:768], b[:768], res, one, zero, 1e-12,
                                   K=512, q_bits=qb, s_q=0.5 if qb == 4 else 0.02, qmin=-8 if qb != 8 else -128,
                                   qmax=7 if qb != 8 else 127)
    lib().mkq_set_small_m_mode(-1)


def part_attn():
    for S, B in ((512, 2), (128, 3)):                    # tcgen05 ping-pong (seq > 128), mma.sync flash
        qkv = (torch.randn(B * S, 3 * 128, device=dev, generator=g) * 0.5).half()
        M.mkq_attention(qkv, 2, B, S, None, mode=M.OUT_I4, s_out=0.05)
        M.mkq_attention(qkv, 2, B, S, None, mode=M.OUT_F32)
    cu = torch.tensor([0, 17, 100, 101, 200], dtype=torch.int32, device=dev)
    qkv = (torch.randn(200, 3 * 128, device=dev, generator=g) * 0.5).half()
    M.mkq_attention(qkv, 2, 4, 128, cu, mode=M.OUT_I4, s_out=0.05)
    q8 = torch.randint(-127, 128, (200, 3 * 128), dtype=torch.int8, device=dev, generator=g)
    M.mkq_attention_i8(q8, 2, 4, 128, 0.01, cu, mode=M.OUT_I4, s_out=0.05)


def part_glue():
    x = torch.randn(300, 1024, device=dev, generator=g)
    M.mkq_quantize_pack(x, torch.tensor([0.5], device=dev), 4, -8, 7)
    M.mkq_quantize_pack(x, torch.tensor([0.02], device=dev), 8, -128, 127)
    M.mkq_absmax_scale(x, 7.0, per_row=True)
    M.mkq_residual_layernorm(x, x, torch.ones(1024, device=dev), torch.zeros(1024, device=dev), 1e-12, bits=4,
                             s_q=0.5)
    M.mkq_fake_quant(x.reshape(-1), torch.tensor([0.5], device=dev), grad_y=torch.ones_like(x.reshape(-1)))
    M.mkq_act_scale(x.reshape(-1), 7.0)
    M.mkq_requant_table(True, 0.3, -8, 7, dev, cache=False)
    M.mkq_interleave_blocks(rnd_u8(2 * 300, 64), 2, 300, 64)


def part_layer():
    h, H, F = 256, 4, 1024
    layers = []
    for i, bits in enumerate((8, 4)):
        p = synth.layer_params(h, H, F, i)
        L = model.build_layer(p, bits, dev)
        model.calibrate(L, torch.from_numpy(synth.activations(128, h, seed=1000000 + i)).to(dev), 2, 64)
        layers.append(L)
    x = torch.from_numpy(synth.hidden_states(2, 64, h, seed=1)).to(dev)
    model.Encoder(layers)(x, 2, 64, out=torch.empty_like(x))
    cu = torch.tensor([0, 100, 160, 300], dtype=torch.int32, device=dev)
    M.mkq_bert_layer(layers[1], torch.from_numpy(synth.hidden_states(1, 300, h, seed=2)).to(dev), 3, 140, cu)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="all")
    a = ap.parse_args()
    for name, fn in (("gemm", part_gemm), ("attn", part_attn), ("glue", part_glue), ("layer", part_layer)):
        if a.part in ("all", name):
            fn()
            torch.cuda.synchronize()
            print(f"{name}: done", flush=True)


if __name__ == "__main__":
    main()
