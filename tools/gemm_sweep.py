"""BASELINE.json configs[4]: W4A4 GEMM shape sweep M = 1..65536 (powers of 2)
x K, N in {768, 1024, 3072, 4096} (272 shapes, fp32 output, bias), against
the int8 tensor and HBM rooflines, with cuBLAS fp32 (TF32 off) and bf16
(torch.matmul) on the same shapes.  Device time: `reps` back-to-back calls
captured in a CUDA graph, CUDA events around 3 replays; weights are
L2-resident for the small shapes (as in a serving step).  Writes gpurun_out/gemm_sweep.{json,md}.

    python tools/gemm_sweep.py [--reps 10] [--quick]
"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2203_13483_b200 import mkq as M


def timeit(fn, reps):
    """Device time per call: `reps` calls captured in one CUDA graph (no host
    launch overhead in the timed region), mean of 3 replays after warm-up."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * reps) * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    pk = bench.peaks()
    int8_peak, hbm = pk["int8_tops_sustained"], pk["hbm_gbs"]
    torch.backends.cuda.matmul.allow_tf32 = False
    dims = [768, 1024, 3072, 4096]
    Ms = [1 << i for i in range(17)] if not a.quick else [1, 128, 4096, 65536]
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    for K in dims:
        w = torch.randint(0, 256, (max(dims), K // 2), generator=g, device="cuda", dtype=torch.uint8)
        wf = torch.randn(max(dims), K, device="cuda")
        wb = wf.bfloat16()
        wi_all = torch.randint(-128, 128, (max(dims), K), device="cuda", dtype=torch.int8)
        for N in dims:
            s_w = torch.full((N,), 1e-3, device="cuda")
            bias = torch.zeros(N, device="cuda")
            for Mm in Ms:
                x = torch.randint(0, 256, (Mm, K // 2), generator=g, device="cuda", dtype=torch.uint8)
                out = torch.empty(Mm, N, device="cuda")
                ours = timeit(lambda: M.mkq_gemm_w4a4(x, w[:N], 0.3, s_w, bias, out=out, K=K), a.reps)
                xf = torch.randn(Mm, K, device="cuda")
                f32 = timeit(lambda: torch.matmul(xf, wf[:N].t()), a.reps)
                xb = xf.bfloat16()
                bf16 = timeit(lambda: torch.matmul(xb, wb[:N].t()), a.reps)
                i8 = None
                try:   # cuBLASLt int8 (torch._int_mm): the practical int8 tensor ceiling
                    if Mm > 16:
                        xi = torch.randint(-128, 128, (Mm, K), device="cuda", dtype=torch.int8)
                        wi = wi_all[:N].t()
                        i8 = timeit(lambda: torch._int_mm(xi, wi), a.reps)
                except Exception:
                    i8 = None
                ops = 2.0 * Mm * N * K
                byts = Mm * K / 2 + N * K / 2 + 4 * Mm * N + 8 * N
                t_tc, t_hbm = ops / (int8_peak * 1e12) * 1e6, byts / (hbm * 1e9) * 1e6
                bound = "tensor" if t_tc >= t_hbm else "hbm"
                rows.append({"M": Mm, "N": N, "K": K, "us": round(ours, 2), "tops": round(ops / ours / 1e6, 1),
                             "frac_int8_peak": round(ops / ours / 1e6 / int8_peak, 4),
                             "gbs": round(byts / ours / 1e3, 1), "bound": bound,
                             "roofline_frac": round(max(t_tc, t_hbm) / ours, 4),
                             "cublas_f32_us": round(f32, 2), "cublas_bf16_us": round(bf16, 2),
                             "cublaslt_int8_us": None if i8 is None else round(i8, 2),
                             "speedup_vs_f32": round(f32 / ours, 2), "speedup_vs_bf16": round(bf16 / ours, 2)})
                del x, out, xf, xb
        print(f"K={K} done", flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "gemm_sweep.json"), "w") as f:
        json.dump({"peaks": pk, "rows": rows}, f)
    lines = ["| M | N | K | ours us | TOPS | frac int8 peak | GB/s | bound | roofline frac | cuBLAS fp32 us | cuBLAS bf16 us | cuBLASLt int8 us | x fp32 | x bf16 |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append("| " + " | ".join(str(r[k]) for k in ("M", "N", "K", "us", "tops", "frac_int8_peak", "gbs", "bound",
                                                           "roofline_frac", "cublas_f32_us", "cublas_bf16_us",
                                                           "cublaslt_int8_us", "speedup_vs_f32", "speedup_vs_bf16")) + " |")
    with open(os.path.join(ROOT, "gpurun_out", "gemm_sweep.md"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
