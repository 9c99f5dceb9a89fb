"""Run the eight launches of one BERT-large W4A4 layer step (bench.py's
workload) once after a warm-up, for ncu captures:

    ncu --set full -k regex:'gemm|attn|ln|quantize' -s <warm-up launches> -c 8 python tools/prof_layer.py
    ncu --metrics gpu__time_duration.sum --csv ... python tools/prof_layer.py --steps 3

--steps N runs N full mkq_bert_layer steps (the bench's timed call) instead.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2203_13483_b200 import mkq as M  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--batch", type=int, default=bench.CFG["batch"])
    a = ap.parse_args()
    bench.CFG["batch"] = a.batch
    dev = torch.device("cuda", 0)
    L, _ = bench.setup_layer(torch, dev, 0)
    B, S, hd = bench.CFG["batch"], bench.CFG["seq"], bench.CFG["hidden"]
    T = B * S
    h_in = torch.from_numpy(synth.hidden_states(B, S, hd, seed=0)).to(dev)
    ws = torch.empty(L.workspace_size(T), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    if a.steps:
        h_out = torch.empty_like(h_in)
        M.mkq_bert_layer(L, h_in, B, S, None, h_out=h_out, ws=ws, stream=stream)   # warm-up
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(a.steps):
            M.mkq_bert_layer(L, h_in, B, S, None, h_out=h_out, ws=ws, stream=stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    else:
        calls, _ = bench.stage_calls(M, L, h_in, B, T, stream)
        for c in calls:       # warm-up pass
            c[1]()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for c in calls:       # profiled pass
            c[1]()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
