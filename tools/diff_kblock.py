import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
def run(env, M, N, K, kb):
    code = f'''
import sys, numpy as np, torch
sys.path.insert(0, "{ROOT}")
from paper_2203_13483_b200 import mkq as M
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randint(0, 256, ({M}, {K}//2), dtype=torch.uint8, device="cuda", generator=g)
W = torch.randint(0, 256, ({N}, {K}//2), dtype=torch.uint8, device="cuda", generator=g)
if {kb} >= 0:
    mask = torch.zeros({K}//2, dtype=torch.bool, device="cuda"); mask[{kb}*64:({kb}+1)*64] = True
    A[:, ~mask] = 0
out = M.mkq_gemm_w4a4(A, W, 1.0, torch.ones({N}, device="cuda"), None, mode=M.OUT_I32, K={K})
torch.cuda.synchronize()
np.save("/tmp/o.npy", out.cpu().numpy())
'''
    subprocess.check_call([sys.executable, "-c", code], env=dict(os.environ, **env))
    return np.load("/tmp/o.npy")
lib = sys.argv[1] if len(sys.argv) > 1 else ""
extra = {"MKQ_LIB": lib} if lib else {}
for kb in [-1] + list(range(8)):
    a = run({"MKQ_GEMM_PATH": "1cta"}, 512, 256, 1024, kb)
    b = run(dict({"MKQ_GEMM_PATH": "2cta", "MKQ_MAX_CLUSTERS": "1"}, **extra), 512, 256, 1024, kb)
    d = np.argwhere(a != b)
    print(f"lib={os.path.basename(lib) or 'default'} kblock={kb}: mismatches {len(d)}"
          + (f" rows {np.unique(d[:,0]//128).tolist()} cols {np.unique(d[:,1]//128).tolist()}" if len(d) else ""), flush=True)
