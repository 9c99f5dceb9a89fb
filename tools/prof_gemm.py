"""Run one W4A4/W8A8 GEMM shape a few times (for ncu captures / quick timing).

    python tools/prof_gemm.py --M 131072 --N 1024 --K 4096 --mode f32 [--bits 4] [--gelu] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2203_13483_b200 import mkq as M  # noqa: E402

MODES = {"f32": M.OUT_F32, "f16": M.OUT_F16, "bf16": M.OUT_BF16, "i32": M.OUT_I32, "i4": M.OUT_I4, "i8": M.OUT_I8}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=131072)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--mode", default="f32")
    ap.add_argument("--gelu", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-table", action="store_true")
    a = ap.parse_args()
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    kb = a.K // 2 if a.bits == 4 else a.K
    A = torch.randint(0, 256, (a.M, kb), dtype=torch.uint8, device=dev, generator=g)
    W = torch.randint(0, 256, (a.N, kb), dtype=torch.uint8, device=dev, generator=g)
    if a.bits == 8:
        A = A.view(torch.int8)
        W = W.view(torch.int8)
    sw = torch.rand(a.N, device=dev) * 1e-3 + 1e-4
    b = torch.rand(a.N, device=dev) * 0.1
    mode = MODES[a.mode]
    fn = M.mkq_gemm_w4a4 if a.bits == 4 else M.mkq_gemm_w8a8
    tab = None if a.no_table else True
    out = fn(A, W, 0.3, sw, b, mode=mode, gelu=a.gelu, s_out=0.05, K=a.K, requant_table=tab,
             qmin=-8 if a.bits == 4 else -128, qmax=7 if a.bits == 4 else 127)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        fn(A, W, 0.3, sw, b, mode=mode, gelu=a.gelu, s_out=0.05, out=out, K=a.K, requant_table=tab,
           qmin=-8 if a.bits == 4 else -128, qmax=7 if a.bits == 4 else 127)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"M={a.M} N={a.N} K={a.K} bits={a.bits} mode={a.mode} gelu={a.gelu} table={not a.no_table}: {ms*1e3:.1f} us, "
          f"{2*a.M*a.N*a.K/ms/1e9:.1f} TOPS")


if __name__ == "__main__":
    main()
