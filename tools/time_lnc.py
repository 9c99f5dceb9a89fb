"""Graph-replayed time of mkq_gemm_residual_ln (small-M N-cluster path vs the
2-CTA kernel via plan mode 0) and of the unfused GEMM + residual_layernorm,
at Table-2 sizes (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_13483_b200 import mkq as M
from paper_2203_13483_b200._lib import lib

def gtime(fn, R=20):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3): fn(st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(R): fn(st)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10): g.replay()
        e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (10 * R)

for Mr, N, K in [(440, 256, 768), (440, 512, 768), (440, 768, 768), (440, 1024, 768), (440, 768, 3072), (128, 768, 768)]:
    a = torch.randint(0, 256, (Mr, K // 2), dtype=torch.uint8, device="cuda")
    w = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda")
    sw = torch.full((N,), 1e-3, device="cuda"); b = torch.zeros(N, device="cuda")
    res = torch.randn(Mr, N, device="cuda"); g1 = torch.ones(N, device="cuda"); z = torch.zeros(N, device="cuda")
    y = torch.empty(Mr, N, device="cuda"); q = torch.empty(Mr, N // 2, dtype=torch.uint8, device="cuda")
    o = torch.empty(Mr, N, device="cuda")
    f = lambda st: M.mkq_gemm_residual_ln(a, w, 0.05, sw, b, res, g1, z, 1e-12, K=K, q_bits=4, s_q=0.5, y=y, q=q, stream=st)
    t_auto = gtime(f)
    lib().mkq_set_small_m_mode(0); t_2cta = gtime(f); lib().mkq_set_small_m_mode(-1)
    def unf(st):
        M.mkq_gemm_w4a4(a, w, 0.05, sw, b, mode=M.OUT_F32, out=o, K=K, stream=st)
        M.mkq_residual_layernorm(o, res, g1, z, 1e-12, bits=4, s_q=0.5, qmin=-8, qmax=7, y=y, q=q, stream=st)
    t_unf = gtime(unf)
    print(f"M={Mr} N={N} K={K}: fused auto {t_auto:.2f} us, fused 2cta {t_2cta:.2f} us, unfused {t_unf:.2f} us", flush=True)
