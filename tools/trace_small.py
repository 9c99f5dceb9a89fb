"""Timeline of the 1-CTA GEMM at Table-2 sizes (diagnostics): builds a
-DMKQ_TTRACE copy of libmkq under build_dbg/ttrace/, runs one GEMM shape
(env SHAPE=M,N,K, BITS, MKQ_SMALL_M=1) and prints per-CTA globaltimer
offsets (us) from the earliest kernel entry.  Slots: 0 entry, 1 setup done,
2 first TMA issued, 3 fifth TMA issued, 4 MMA first stage ready,
5 MMA last stage ready, 6 epilogue acc ready, 7 partial staged,
8 thread 128's reduce/epilogue done, 9 exit, 10..15 MMA stage 2..7 ready."""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_13483_b200 import build as B
extra = os.environ.get("EXTRA", "").split()   # e.g. EXTRA=-DMKQ_ABL_NOSTORE (ablation builds)
dbg = os.path.join(ROOT, "build_dbg", "ttrace" + "".join(f.replace("-D", "_") for f in extra), "libmkq.so")
if not os.environ.get("NO_BUILD"):
    os.makedirs(os.path.dirname(dbg), exist_ok=True)
    subprocess.check_call([B.NVCC, *B.FLAGS, "-DMKQ_TTRACE", *extra, "-o", dbg, os.path.join(B.CSRC, "mkq_abi.cu"), "-ldl"])
if os.environ.get("BUILD_ONLY"):
    sys.exit(0)
os.environ["MKQ_LIB"] = dbg
import numpy as np, torch
from paper_2203_13483_b200 import mkq as M
from paper_2203_13483_b200._lib import lib
Mm, N, K = (int(v) for v in os.environ.get("SHAPE", "440,768,768").split(","))
bits = int(os.environ.get("BITS", 4))
g = torch.Generator().manual_seed(0)
kb = K // 2 if bits == 4 else K
a = torch.randint(0, 256, (Mm, kb), generator=g, dtype=torch.uint8).cuda()
w = torch.randint(0, 256, (N, kb), generator=g, dtype=torch.uint8).cuda()
if bits == 8:
    a, w = a.view(torch.int8), w.view(torch.int8)
sw = torch.full((N,), 1e-3, device="cuda"); b = torch.zeros(N, device="cuda")
gemm = M.mkq_gemm_w4a4 if bits == 4 else M.mkq_gemm_w8a8
if os.environ.get("FUSED_LN"):   # the small-M fused GEMM + residual + LN (slots 12-15: LN pass 2)
    res = torch.randn(Mm, N, device="cuda"); g1 = torch.ones(N, device="cuda")
    def gemm(a, w, s_a, sw, b, K, out=None):
        return M.mkq_gemm_residual_ln(a, w, s_a, sw, b, res, g1, b, 1e-12, K=K, q_bits=4, s_q=0.5)
out = gemm(a, w, 0.3, sw, b, K=K)
buf = torch.zeros(256 * 16 * 2, dtype=torch.int64, device="cuda")
lib().mkq_debug_set_ttrace.argtypes = [ctypes.c_void_p]
for rep in range(3):
    buf.zero_()
    assert lib().mkq_debug_set_ttrace(ctypes.c_void_p(buf.data_ptr())) == 0
    torch.cuda.synchronize()
    gemm(a, w, 0.3, sw, b, K=K, out=out)
    torch.cuda.synchronize()
tr = buf.view(256, 16, 2).cpu().numpy()
used = [c for c in range(256) if tr[c, 0, 0]]
t0 = min(tr[c, 0, 0] for c in used)
print(f"shape {Mm}x{N}x{K} bits {bits}: {len(used)} CTAs")
for c in used[:6] + used[-3:]:
    print(f"cta {c:3d}: " + " ".join(f"{s}:{(tr[c, s, 0] - t0) / 1e3:6.2f}" if tr[c, s, 0] else f"{s}:  -   " for s in range(16)))
ends = sorted((tr[c, 9, 0] - t0) / 1e3 for c in used)
starts = sorted((tr[c, 0, 0] - t0) / 1e3 for c in used)
print("entry spread us: %.2f..%.2f  exit spread us: %.2f..%.2f" % (starts[0], starts[-1], ends[0], ends[-1]))
