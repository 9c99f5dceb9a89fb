"""Small-M GEMMs of the Table-2 layer (M = 440) for ncu source-level captures:
QKV (N 2304, K 768, fp16 out) and FFN2 (N 768, K 3072, fp32 out, K split over a cluster)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_13483_b200 import mkq as M
g = torch.Generator(device="cuda").manual_seed(0)
for (Mm, N, K, mode) in ((440, 2304, 768, M.OUT_F16), (440, 768, 3072, M.OUT_F32)):
    a = torch.randint(0, 256, (Mm, K // 2), generator=g, device="cuda", dtype=torch.uint8)
    w = torch.randint(0, 256, (N, K // 2), generator=g, device="cuda", dtype=torch.uint8)
    sw = torch.full((N,), 1e-3, device="cuda"); b = torch.zeros(N, device="cuda")
    for _ in range(3):
        M.mkq_gemm_w4a4(a, w, 0.3, sw, b, mode=mode, K=K)
torch.cuda.synchronize()
