"""Device time of the short-sequence attention kernels at Table-2 sizes
(graph-replayed): fp16 mma.sync flash kernel vs the NEXT(2) integer core."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2203_13483_b200 import mkq as M


def timeit(fn, reps=20):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); g.replay(); e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for bs, valid in ((16, 440), (16, 681), (64, 2298), (32, 4096)):
    H = 12
    lens = synth.varlen_seqlens(bs, valid, 128, seed=bs + valid) if valid != 4096 else np.full(32, 128)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), device="cuda")
    qkv16 = (torch.randn(valid, 3 * 768, device="cuda") * 0.5).half()
    qkv8 = torch.randint(-127, 128, (valid, 3 * 768), device="cuda", dtype=torch.int8)
    t16 = timeit(lambda: M.mkq_attention(qkv16, H, bs, 128, cu, mode=M.OUT_I4, s_out=0.05))
    t8 = timeit(lambda: M.mkq_attention_i8(qkv8, H, bs, 128, 0.02, cu, mode=M.OUT_I4, s_out=0.05))
    t8b = timeit(lambda: M.mkq_attention_i8(qkv8, H, bs, 128, 0.2, cu, mode=M.OUT_I4, s_out=0.05))
    print(f"bs={bs} tokens={valid} max_len={int(max(lens))}: fp16 {t16:.1f} us, int8 {t8:.1f} us (flat scores), "
          f"{t8b:.1f} us (peaked scores)")
