"""Event timeline of CTA 0 of the 2-CTA W4A4 GEMM on the FFN1 shape (diagnostics).
Builds a -DMKQ_GTRACE copy of libmkq under build_dbg/gtrace/, runs FFN1 of the
bench layer and prints per-warp time splits between consecutive tags.
Tags: epilogue 1 scales loaded, 2 staged, 3 tfull ok, 4 staging free, 5 TMEM
loaded, 6 codes done, 8 tempty arrived; MMA 29/30 tempty wait, 31 full8 ok;
unpack 19/20 fullP wait, 21 empty8 ok."""
import collections, ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_13483_b200 import build as B
dbg = os.path.join(ROOT, "build_dbg", "gtrace", "libmkq.so")
if not os.environ.get("NO_BUILD"):
    os.makedirs(os.path.dirname(dbg), exist_ok=True)
    subprocess.check_call([B.NVCC, *B.FLAGS, "-DMKQ_GTRACE", "-o", dbg, os.path.join(B.CSRC, "mkq_abi.cu"), "-ldl"])
if os.environ.get("BUILD_ONLY"):
    sys.exit(0)
os.environ["MKQ_LIB"] = dbg
import torch
import bench, synth
from paper_2203_13483_b200 import mkq as M
from paper_2203_13483_b200._lib import lib
dev = torch.device("cuda", 0)
L, _ = bench.setup_layer(torch, dev, 0)
Bn, S, hd = bench.CFG["batch"], bench.CFG["seq"], bench.CFG["hidden"]
T = Bn * S
h_in = torch.from_numpy(synth.hidden_states(Bn, S, hd, seed=0)).to(dev)
ws = torch.empty(L.workspace_size(T), dtype=torch.uint8, device=dev)
calls, _ = bench.stage_calls(M, L, h_in, Bn, T, torch.cuda.current_stream())
for c in calls:
    c[1]()
name = os.environ.get("STAGE", "gemm_ffn1")
fn = [c[1] for c in calls if c[0] == name][0]
slots = 512
buf = torch.zeros(48 * slots * 2, dtype=torch.int64, device="cuda")
lib().mkq_debug_set_gtrace.argtypes = [ctypes.c_void_p]
assert lib().mkq_debug_set_gtrace(ctypes.c_void_p(buf.data_ptr())) == 0
torch.cuda.synchronize()
fn()
torch.cuda.synchronize()
tr = buf.view(48, slots, 2).cpu().numpy()
t0 = min(int(tr[w, 0, 1]) for w in range(24) if tr[w, 0, 1])  # CTA 0 clock (CTA 1: separate SM clock)
for w in [1] + list(range(4, 24)) + list(range(24 + 4, 48)):
    ev = [(int(a), int(b)) for a, b in tr[w] if b]
    if not ev:
        continue
    acc = collections.Counter()
    for (a, ta), (b, tb) in zip(ev, ev[1:]):
        acc[f"{a}->{b}"] += tb - ta
    tot = ev[-1][1] - ev[0][1] or 1
    print(f"warp {w:2d} n={len(ev)} span {tot}: " + ", ".join(f"{k}:{100*v/tot:.0f}%" for k, v in acc.most_common(7)))
print("warp 4 first events:", " ".join(f"{a}@{b - t0}" for a, b in [(int(a), int(b)) for a, b in tr[4] if b][:40]))
print("warp 1 first events:", " ".join(f"{a}@{b - t0}" for a, b in [(int(a), int(b)) for a, b in tr[1] if b][:40]))
# per-warp averages: chunk compute (5->6), tfull wait (2->3), tile period (1->1)
import numpy as np
for w in list(range(4, 20)) + list(range(28, 44)):
    ev = [(int(a), int(b)) for a, b in tr[w] if b]
    comp = [tb - ta for (a, ta), (b, tb) in zip(ev, ev[1:]) if (a, b) == (5, 6)]
    wait = [tb - ta for (a, ta), (b, tb) in zip(ev, ev[1:]) if (a, b) == (2, 3)]
    t1 = [t for a, t in ev if a == 1]
    per = np.diff(t1)
    print(f"warp {w:2d} smsp {w % 4}: compute/chunk {np.mean(comp):6.0f}  tfull-wait {np.mean(wait):6.0f}  tile period {np.mean(per):6.0f}")
