"""Paper Table-2 BERT-base layer (BS 16, 440 valid tokens by default; env BITS, T,
BS) through mkq_bert_layer, for ncu captures limited to the profiler region
(--profile-from-start off): 3 steps (launch list), --once 1 step (--set full)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2203_13483_b200 import mkq as M, model
bits = int(os.environ.get("BITS", 4)); T = int(os.environ.get("T", 440)); bs = int(os.environ.get("BS", 16))
h, H, F, S = 768, 12, 3072, 128
p = synth.layer_params(h, H, F, 0)
L = model.build_layer(p, bits, "cuda")
model.calibrate(L, torch.from_numpy(synth.hidden_states(8, S, h, seed=1000000)).cuda(), 8, S)
lens = synth.varlen_seqlens(bs, T, S, seed=bs + T)
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), device="cuda")
x = torch.from_numpy(synth.hidden_states(1, T, h, seed=1)).cuda()
out = torch.empty_like(x)
ws = torch.zeros(L.workspace_size(T), dtype=torch.uint8, device="cuda")
for _ in range(3):
    M.mkq_bert_layer(L, x, bs, S, cu, h_out=out, ws=ws)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(1 if "--once" in sys.argv else 3):
    M.mkq_bert_layer(L, x, bs, S, cu, h_out=out, ws=ws)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("fused LN:", L.fused_ln(T))
