"""One launch each of the QAT / calibration kernels on the bench's layer
input shape (131072 x 1024 fp32), for ncu captures (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_13483_b200 import mkq as M
x = torch.randn(131072, 1024, device="cuda")
gy = torch.randn_like(x)
sc = torch.tensor([0.5558], device="cuda")
for _ in range(2):
    M.mkq_fake_quant(x, sc, -8, 7, grad_y=gy)
    M.mkq_act_scale(x, 7.0, 0.9999)
torch.cuda.synchronize()
