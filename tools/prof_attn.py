"""Time mkq_attention alone at BERT-large b256 s512 (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_13483_b200 import mkq as M
B, S, H = int(os.environ.get("B", 256)), 512, 16
T, hd = B * S, H * 64
qkv = (torch.randn(T, 3 * hd, device="cuda") * 0.8).half()
out = torch.empty(T, hd // 2, dtype=torch.uint8, device="cuda")
for _ in range(2):
    M.mkq_attention(qkv, H, B, S, None, mode=M.OUT_I4, s_out=0.05, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    M.mkq_attention(qkv, H, B, S, None, mode=M.OUT_I4, s_out=0.05, out=out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"attention path={os.environ.get('MKQ_ATTN','pp')} B={B}: {ms*1e3:.1f} us, {4*T*S*hd/ms/1e9:.1f} TFLOP/s")
if os.environ.get("KNAMES"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        M.mkq_attention(qkv, H, B, S, None, mode=M.OUT_I4, s_out=0.05, out=out)
        torch.cuda.synchronize()
    for e in prof.key_averages():
        print("KERNEL", e.key[:80], e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
