"""Event timeline of the ping-pong attention kernel's CTA 0 (diagnostics).

Builds a -DMKQ_TRACE copy of libmkq under build_dbg/, runs one attention call
at BERT-large b256 s512 and prints per-warp (tag, clock) events relative to
the first one.  Tags: softmax 1 wait-S start, 2 S ready, 3 max done, 4 XU
turn acquired, 5 P handed to MMA, 6/7 O wait; MMA 10/11 wait P_A, 20/21
wait P_B, 30 block done.
"""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_13483_b200 import build as B
dbg = os.environ.get("TRACE_LIB") or os.path.join(ROOT, "build_dbg", "libmkq.so")
if not os.environ.get("NO_BUILD"):
    os.makedirs(os.path.dirname(dbg), exist_ok=True)
    extra = os.environ.get("EXTRA_FLAGS", "").split()
    subprocess.check_call([B.NVCC, *B.FLAGS, "-DMKQ_TRACE", *extra, "-o", dbg, os.path.join(B.CSRC, "mkq_abi.cu"), "-ldl"])
os.environ["MKQ_LIB"] = dbg
import torch
from paper_2203_13483_b200 import mkq as M
from paper_2203_13483_b200._lib import lib

Bn, S, H = int(os.environ.get("B", 256)), 512, 16
T, hd = Bn * S, H * 64
qkv = (torch.randn(T, 3 * hd, device="cuda") * 0.8).half()
out = torch.empty(T, hd // 2, dtype=torch.uint8, device="cuda")
M.mkq_attention(qkv, H, Bn, S, None, mode=M.OUT_I4, s_out=0.05, out=out)
slots = 512
NW = 12   # warps per CTA (attention_pp_sm100.cuh kThreads / 32)
buf = torch.zeros(NW * slots * 2, dtype=torch.int64, device="cuda")
assert lib().mkq_debug_set_trace(ctypes.c_void_p(buf.data_ptr())) == 0
torch.cuda.synchronize()
M.mkq_attention(qkv, H, Bn, S, None, mode=M.OUT_I4, s_out=0.05, out=out)
torch.cuda.synchronize()
tr = buf.view(NW, slots, 2).cpu().numpy()
t0 = min(int(tr[w, 0, 1]) for w in range(NW) if tr[w, 0, 1])
nshow = int(os.environ.get("N", 60))
for w in [int(x) for x in os.environ.get("WARPS", "1,4,8").split(",")]:
    ev = [(int(a), int(b) - t0) for a, b in tr[w] if b]
    print(f"warp {w}: {len(ev)} events")
    print("  " + " ".join(f"{a}@{b}" for a, b in ev[:nshow]))
# summary: per-softmax-warp time split
import collections
for w in range(4, NW):
    ev = [(int(a), int(b)) for a, b in tr[w] if b]
    acc = collections.Counter()
    for (a, ta), (b, tb) in zip(ev, ev[1:]):
        acc[f"{a}->{b}"] += tb - ta
    tot = ev[-1][1] - ev[0][1] if ev else 1
    print(f"warp {w} span {tot}: " + ", ".join(f"{k}:{100*v/tot:.0f}%" for k, v in acc.most_common(6)))
