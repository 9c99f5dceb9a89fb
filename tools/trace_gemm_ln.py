"""Event timeline of CTA 0 of the fused GEMM + residual + LN kernel at the
C4 O-projection shape (diagnostics; -DMKQ_GTRACE build under build_dbg/gtrace).
Tags (epilogue warps): 40 tile start, 41 residual TMA issued, 42 accumulator
ready, 43 pass 1 done (TMEM released), 44 local stats, 45 quadrant barrier,
46 partial published, 47 group statistics arrived, 48 output issued;
MMA 29/30 tempty wait, 31 full8; unpack 19/20 fullP, 21 empty8."""
import collections, ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_13483_b200 import build as B
dbg = os.path.join(ROOT, "build_dbg", "gtrace", "libmkq.so")
if not os.environ.get("NO_BUILD"):
    os.makedirs(os.path.dirname(dbg), exist_ok=True)
    subprocess.check_call([B.NVCC, *B.FLAGS, "-DMKQ_GTRACE", "-o", dbg, os.path.join(B.CSRC, "mkq_abi.cu"), "-ldl"])
os.environ["MKQ_LIB"] = dbg
import torch
from paper_2203_13483_b200 import mkq as M
from paper_2203_13483_b200._lib import lib
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
Mr, N, K = int(os.environ.get("M", 131072)), 1024, int(os.environ.get("K", 1024))
A = torch.randint(0, 256, (Mr, K // 2), dtype=torch.uint8, device=dev, generator=g)
W = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev, generator=g)
sw = torch.rand(N, device=dev) * 1e-4 + 1e-4
b = torch.rand(N, device=dev) * 0.1
res = torch.randn(Mr, N, device=dev)
one, zero = torch.ones(N, device=dev), torch.zeros(N, device=dev)
fn = lambda: M.mkq_gemm_residual_ln(A, W, 0.05, sw, b, res, one, zero, 1e-12, K=K, q_bits=4, s_q=0.5)  # noqa
fn()
slots = 512
buf = torch.zeros(48 * slots * 2, dtype=torch.int64, device="cuda")
lib().mkq_debug_set_gtrace.argtypes = [ctypes.c_void_p]
assert lib().mkq_debug_set_gtrace(ctypes.c_void_p(buf.data_ptr())) == 0
torch.cuda.synchronize()
fn()
torch.cuda.synchronize()
tr = buf.view(48, slots, 2).cpu().numpy()
t0 = min(int(tr[w, 0, 1]) for w in range(24) if tr[w, 0, 1])
for w in [1, 4, 5, 8, 11] + list(range(12, 16)):
    ev = [(int(a), int(b)) for a, b in tr[w] if b]
    if not ev:
        continue
    acc = collections.Counter()
    for (a, ta), (b2, tb) in zip(ev, ev[1:]):
        acc[f"{a}->{b2}"] += tb - ta
    tot = ev[-1][1] - ev[0][1] or 1
    print(f"warp {w:2d} n={len(ev)} span {tot}: " + ", ".join(f"{k}:{100*v/tot:.0f}%" for k, v in acc.most_common(9)))
for w in (4,):
    print(f"warp {w} first events:", " ".join(f"{a}@{b2 - t0}" for a, b2 in [(int(a), int(b)) for a, b in tr[w] if b][:90]))
