"""Validity flags of the requant tables (general / compact int4) for the
FFN2-input scales the layer calibration produces (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2203_13483_b200 import mkq as M, model
from paper_2203_13483_b200.mkq import mkq_requant_table
h, H, F, S = 768, 12, 3072, 128
p = synth.layer_params(h, H, F, 0)
L = model.build_layer(p, 4, "cuda")
model.calibrate(L, torch.from_numpy(synth.hidden_states(8, S, h, seed=1000000)).cuda(), 8, S)
def flags(s):
    t = mkq_requant_table(True, s, -8, 7, "cuda", cache=False).cpu().numpy()
    gen_valid = int(t[28:32].view(np.int32)[0])          # Header.valid (offset 28)
    off4 = 64 + 1024 * 8
    return gen_valid, int(t[off4 + 8:off4 + 12].view(np.int32)[0])   # Header4.valid (offset 8)
print("bert-base calibrated s_ffn2_in", L.scales["s_ffn2_in"], "valid(general, compact)", flags(L.scales["s_ffn2_in"]))
bad = 0
ss = np.geomspace(0.005, 0.5, 400).astype(np.float32)
res = [flags(float(s)) for s in ss]
print("sweep s in [0.005, 0.5] (400 pts): general invalid", sum(1 for g, c in res if not g), "compact invalid", sum(1 for g, c in res if not c))
print("compact-invalid s:", [float(s) for s, (g, c) in zip(ss, res) if not c][:40])
