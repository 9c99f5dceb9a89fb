"""One launch of the NEXT(2) integer attention kernel (32 x 128 tokens, 12 heads) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_13483_b200 import mkq as M
qkv8 = torch.randint(-127, 128, (4096, 3 * 768), device="cuda", dtype=torch.int8)
for _ in range(2):
    M.mkq_attention_i8(qkv8, 12, 32, 128, 0.02, None, mode=M.OUT_I4, s_out=0.05)
torch.cuda.synchronize()
