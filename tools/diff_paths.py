"""Compare the 2-CTA W4A4 path against the 1-CTA path on one shape (diagnostics)."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def run(path, M, N, K, mode):
    code = f'''
import os, sys, numpy as np, torch
sys.path.insert(0, "{os.path.dirname(os.path.dirname(os.path.abspath(__file__)))}")
from paper_2203_13483_b200 import mkq as M
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randint(0, 256, ({M}, {K}//2), dtype=torch.uint8, device="cuda", generator=g)
W = torch.randint(0, 256, ({N}, {K}//2), dtype=torch.uint8, device="cuda", generator=g)
sw = torch.ones({N}, device="cuda")
out = M.mkq_gemm_w4a4(A, W, 1.0, sw, None, mode=M.OUT_I32, K={K})
torch.cuda.synchronize()
np.save("/tmp/out_{path}.npy", out.cpu().numpy())
'''
    env = dict(os.environ, MKQ_GEMM_PATH=path)
    subprocess.check_call([sys.executable, "-c", code], env=env)
    return np.load(f"/tmp/out_{path}.npy")

M_, N_, K_ = [int(v) for v in sys.argv[1:4]]
a = run("1cta", M_, N_, K_, 0)
b = run("2cta", M_, N_, K_, 0)
d = np.argwhere(a != b)
print("mismatches", len(d), "of", a.size)
if len(d):
    r, c = d[:, 0], d[:, 1]
    print("rows: min", r.min(), "max", r.max(), "unique tiles(256)", np.unique(r // 256)[:20], "n", len(np.unique(r // 256)))
    print("row%256 hist", np.bincount(r % 256 // 32, minlength=8))
    print("cols: unique n-tiles(256)", np.unique(c // 256)[:20], "col%256 hist", np.bincount(c % 256 // 32, minlength=8))
    print("sample", [(int(x), int(y), int(a[x, y]), int(b[x, y])) for x, y in d[:10]])
