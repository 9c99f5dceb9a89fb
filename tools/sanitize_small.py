"""Small invocations of every kernel for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2203_13483_b200 import mkq as M, model
dev = "cuda"
h, H, F = 128, 2, 512
p = synth.layer_params(h, H, F, 0)
for bits in (4, 8):
    L = model.build_layer(p, bits, dev)
    model.calibrate(L, torch.from_numpy(synth.activations(128, h, seed=1000000)).to(dev), 2, 64)
    x = torch.from_numpy(synth.hidden_states(1, 300, h, seed=1)).to(dev)
    cu = torch.tensor([0, 100, 160, 300], dtype=torch.int32, device=dev)
    M.mkq_bert_layer(L, x, 3, 140, cu)
# 2-CTA GEMM with ragged M, both warp configs, all modes
A = torch.randint(0, 256, (300, 512), dtype=torch.uint8, device=dev)
W = torch.randint(0, 256, (512, 512), dtype=torch.uint8, device=dev)
sw = torch.rand(512, device=dev) * 1e-3 + 1e-4
for mode in (M.OUT_F32, M.OUT_F16, M.OUT_I4, M.OUT_I8, M.OUT_I32):
    M.mkq_gemm_w4a4(A, W, 0.3, sw, None, mode=mode, gelu=mode in (M.OUT_I4,), s_out=0.05,
                    qmin=-8 if mode != M.OUT_I8 else -128, qmax=7 if mode != M.OUT_I8 else 127, K=1024)
    M.mkq_gemm_w4a4(A, W, 0.3, sw, None, mode=mode, s_out=0.05, qmin=-8 if mode != M.OUT_I8 else -128,
                    qmax=7 if mode != M.OUT_I8 else 127, K=1024)
torch.cuda.synchronize()
print("sanitize workload done")
