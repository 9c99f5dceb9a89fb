"""Per-stage CUDA-event times of bench.py's layer step (diagnostics; for
ablation builds selected with MKQ_LIB=...).   python tools/stage_times.py [--reps 10] [--only gemm_ffn1,...]"""
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    L, _ = bench.setup_layer(torch, dev, 0)
    B, S, hd = bench.CFG["batch"], bench.CFG["seq"], bench.CFG["hidden"]
    T = B * S
    h_in = torch.from_numpy(synth.hidden_states(B, S, hd, seed=0)).to(dev)
    ws = torch.empty(L.workspace_size(T), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    calls, _ = bench.stage_calls(M, L, h_in, B, T, stream)
    for c in calls:
        c[1]()
    torch.cuda.synchronize()
    only = set(a.only.split(",")) if a.only else None
    out = []
    for name, fn, ops in calls:
        if only and name not in only:
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.reps * 1e3
        out.append(f"{name}={us:.1f}us" + (f"({ops / us / 1e6:.0f}TOPS)" if ops else ""))
    print(os.environ.get("MKQ_LIB", "libmkq.so"), " ".join(out))


if __name__ == "__main__":
    main()
