"""Diagnostics: 2-CTA vs 1-CTA on small shapes with a capped cluster count."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def run(env, M, N, K, seed=0):
    code = f'''
import sys, numpy as np, torch
sys.path.insert(0, "{ROOT}")
from paper_2203_13483_b200 import mkq as M
g = torch.Generator(device="cuda").manual_seed({seed})
A = torch.randint(0, 256, ({M}, {K}//2), dtype=torch.uint8, device="cuda", generator=g)
W = torch.randint(0, 256, ({N}, {K}//2), dtype=torch.uint8, device="cuda", generator=g)
out = M.mkq_gemm_w4a4(A, W, 1.0, torch.ones({N}, device="cuda"), None, mode=M.OUT_I32, K={K})
torch.cuda.synchronize()
np.save("/tmp/o.npy", out.cpu().numpy())
'''
    subprocess.check_call([sys.executable, "-c", code], env=dict(os.environ, **env))
    return np.load("/tmp/o.npy")

for (Mm, N, K, cl) in [(512, 256, 128, 1), (512, 256, 256, 1), (512, 256, 1024, 1), (256, 512, 128, 1),
                       (1024, 256, 128, 1), (1024, 256, 128, 2), (768, 256, 512, 1)]:
    a = run({"MKQ_GEMM_PATH": "1cta"}, Mm, N, K)
    b = run({"MKQ_GEMM_PATH": "2cta", "MKQ_MAX_CLUSTERS": str(cl)}, Mm, N, K)
    d = np.argwhere(a != b)
    msg = f"M={Mm} N={N} K={K} clusters={cl}: mismatches {len(d)}/{a.size}"
    if len(d):
        tiles = np.unique((d[:, 0] // 256) * (N // 256) + d[:, 1] // 256)
        msg += f" tiles={tiles.tolist()} rows%256 hist={np.bincount(d[:,0]%256//32, minlength=8).tolist()}"
        r, c = d[0]
        msg += f" first=({r},{c}) {a[r,c]} vs {b[r,c]}"
    print(msg, flush=True)
