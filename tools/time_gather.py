"""Time the fused all-gather FFN1 GEMM (mkq_gemm_w4a4_gather) against the
unfused per-rank GEMM + interleave of the gathered blocks, on one GPU with
every simulated rank's buffer local (so it measures the extra epilogue
stores and the counter protocol, not NVLink)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_13483_b200 import mkq as M  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    T, K, F = 16384, 1024, 4096
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(0, 256, (T, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    tab = M.mkq_requant_table(True, 0.05, -8, 7, "cuda")
    for world in (1, 2, 4, 8):
        Fl = F // world
        w = torch.randint(0, 256, (Fl, K // 2), dtype=torch.uint8, device="cuda", generator=g)
        s_w = torch.full((Fl,), 2e-3, device="cuda")
        b = torch.zeros(Fl, device="cuda")
        bufs = [torch.empty((T, F // 2), dtype=torch.uint8, device="cuda") for _ in range(world)]
        cnt = torch.zeros((world, 64), dtype=torch.int32, device="cuda")
        blocks = torch.empty((world, T, Fl // 2), dtype=torch.uint8, device="cuda")

        def plain():
            M.mkq_gemm_w4a4(a, w, 0.3, s_w, b, mode=M.OUT_I4, gelu=True, s_out=0.05, K=K, out=blocks[0],
                            requant_table=tab)

        def plain_il():
            plain()
            M.mkq_interleave_blocks(blocks, world, T, Fl // 2)

        def fused():
            M.mkq_gemm_w4a4_gather(a, w, 0.3, s_w, b, [t.data_ptr() for t in bufs],
                                   [cnt[i].data_ptr() for i in range(world)], col0=0, ldo=F // 2, s_out=0.05, K=K,
                                   requant_table=tab)

        tp, ti, tf = timeit(plain), timeit(plain_il), timeit(fused)
        print(f"world={world} N={Fl}: gemm {tp:.1f} us, gemm+interleave {ti:.1f} us, "
              f"fused gather ({world} buffers) {tf:.1f} us")


if __name__ == "__main__":
    main()
