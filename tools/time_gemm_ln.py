"""Timing (diagnostics): fused mkq_gemm_residual_ln vs the unfused
GEMM (fp32) + mkq_residual_layernorm at the BERT-large C4 shapes
(O-projection + LN1 with int4 codes; FFN2 + LN2).   python tools/time_gemm_ln.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_13483_b200 import mkq as M  # noqa: E402


def ev(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    Mr = int(os.environ.get("M", 131072))
    for name, N, K, qb in (("o_proj+ln1", 1024, 1024, 4), ("ffn2+ln2", 1024, 4096, 0)):
        A = torch.randint(0, 256, (Mr, K // 2), dtype=torch.uint8, device=dev, generator=g)
        W = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev, generator=g)
        sw = torch.rand(N, device=dev) * 1e-4 + 1e-4
        b = torch.rand(N, device=dev) * 0.1
        res = torch.randn(Mr, N, device=dev)
        gam = torch.ones(N, device=dev)
        bet = torch.zeros(N, device=dev)
        y = torch.empty(Mr, N, device=dev)
        q = torch.empty(Mr, N // 2, dtype=torch.uint8, device=dev)
        o = torch.empty(Mr, N, device=dev)
        fused = ev(lambda: M.mkq_gemm_residual_ln(A, W, 0.05, sw, b, res, gam, bet, 1e-12, K=K, q_bits=qb, s_q=0.5,
                                                  y=y, q=q if qb else None))
        t_g = ev(lambda: M.mkq_gemm_w4a4(A, W, 0.05, sw, b, mode=M.OUT_F32, out=o, K=K))
        t_l = ev(lambda: M.mkq_residual_layernorm(o, res, gam, bet, 1e-12, bits=qb, s_q=0.5, y=y,
                                                   q=q if qb else None))
        ops = 2.0 * Mr * N * K
        print(f"{name}: fused {fused:.1f} us ({ops / fused / 1e6:.0f} TOPS) vs gemm {t_g:.1f} + ln {t_l:.1f} = "
              f"{t_g + t_l:.1f} us")


if __name__ == "__main__":
    main()
