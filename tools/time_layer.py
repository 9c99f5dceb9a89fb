"""CUDA-event time of bench.py's C4 layer step (mkq_bert_layer), mean of 10 (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2203_13483_b200 import mkq as M
dev = torch.device("cuda", 0)
L, _ = bench.setup_layer(torch, dev, 0)
B, S, hd = bench.CFG["batch"], bench.CFG["seq"], bench.CFG["hidden"]
h_in = torch.from_numpy(synth.hidden_states(B, S, hd, seed=0)).to(dev)
ws = torch.empty(L.workspace_size(B * S), dtype=torch.uint8, device=dev)
out = torch.empty_like(h_in)
for _ in range(3): M.mkq_bert_layer(L, h_in, B, S, None, h_out=out, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): M.mkq_bert_layer(L, h_in, B, S, None, h_out=out, ws=ws)
e1.record(); torch.cuda.synchronize()
print(f"MKQ_PDL_ROWS={os.environ.get('MKQ_PDL_ROWS', 'default')}: layer {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
