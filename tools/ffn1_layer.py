"""Run the bench layer's FFN1 GEMM (GELU + int4 requant, calibrated scales and
real-layer inputs) a few times, for ncu captures (diagnostics).
    python tools/ffn1_layer.py [--reps 3] [--stage gemm_ffn1]"""
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--stage", default="gemm_ffn1")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    L, _ = bench.setup_layer(torch, dev, 0)
    B, S, hd = bench.CFG["batch"], bench.CFG["seq"], bench.CFG["hidden"]
    h_in = torch.from_numpy(synth.hidden_states(B, S, hd, seed=0)).to(dev)
    stream = torch.cuda.current_stream()
    calls, _ = bench.stage_calls(M, L, h_in, B, B * S, stream)
    names = [c[0] for c in calls]
    k = names.index(a.stage)
    for c in calls[:k]:      # produce the stage's real inputs
        c[1]()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()   # ncu --profile-from-start off captures only these launches
    for _ in range(a.reps):
        calls[k][1]()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", a.stage)


if __name__ == "__main__":
    main()
