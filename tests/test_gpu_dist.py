"""Column-parallel FFN on one GPU, ranks simulated in sequence: the per-rank
column blocks, reassembled with mkq_interleave_blocks (what the NCCL
all-gather feeds), reproduce the single-GPU FFN + LN2 bit-exactly."""
import numpy as np
import pytest
import torch

import oracle
from oracle import layer as OL
import synth

pytestmark = pytest.mark.gpu

from paper_2203_13483_b200 import dist as D  # noqa: E402
from paper_2203_13483_b200 import mkq as M  # noqa: E402
from paper_2203_13483_b200 import model  # noqa: E402

DEV = "cuda:0"


@pytest.mark.parametrize("bits,world", [(4, 2), (4, 4), (8, 2)])
def test_column_parallel_ffn_matches_single_gpu(bits, world):
    hidden, heads, ffn = 256, 4, 1024
    p = synth.layer_params(hidden, heads, ffn, 0)
    L = model.build_layer(p, bits, DEV)
    T = 300
    h1 = torch.from_numpy(synth.activations(T, hidden, seed=4)).to(DEV)
    model.calibrate(L, torch.from_numpy(synth.activations(128, hidden, seed=1000000)).to(DEV), 2, 64)
    lo, hi = model.act_range(bits)
    codes = M.mkq_quantize_pack(h1, torch.tensor([L.scales["s_ffn1_in"]], device=DEV), bits, lo, hi)
    gemm = M.mkq_gemm_w4a4 if bits == 4 else M.mkq_gemm_w8a8
    t = L.t
    a2 = gemm(codes, t["w_1"], L.scales["s_ffn1_in"], t["sw_1"], t["b_1"], mode=M.OUT_I4 if bits == 4 else M.OUT_I8,
              gelu=True, s_out=L.scales["s_ffn2_in"], qmin=lo, qmax=hi, K=hidden)
    f = gemm(a2, t["w_2"], L.scales["s_ffn2_in"], t["sw_2"], t["b_2"], mode=M.OUT_F32, K=ffn)
    ref = M.mkq_residual_layernorm(f, h1, t["ln2_g"], t["ln2_b"], L.ln_eps)

    parts = [D.ColumnParallelFFN(L, r, world) for r in range(world)]
    a_blocks = torch.stack([pp.ffn1_local(codes) for pp in parts])
    a_full = M.mkq_interleave_blocks(a_blocks, world, T, a_blocks.shape[2])
    if bits == 8:
        a_full = a_full.view(torch.int8)
    assert torch.equal(a_full.view(torch.uint8), a2.view(torch.uint8))
    f_blocks = torch.stack([pp.ffn2_local(a_full) for pp in parts])
    f_full = M.mkq_interleave_blocks(f_blocks.view(torch.uint8), world, T, parts[0].hl * 4).view(torch.float32)
    assert torch.equal(f_full, f)
    out = M.mkq_residual_layernorm(f_full, h1, t["ln2_g"], t["ln2_b"], L.ln_eps)
    assert torch.equal(out, ref)


def test_interleave_blocks_against_reference():
    g, rows, cb = 3, 257, 48
    src = torch.randint(0, 256, (g, rows, cb), dtype=torch.uint8, device=DEV)
    out = M.mkq_interleave_blocks(src, g, rows, cb)
    assert torch.equal(out, D.interleave_reference(src))


def _cp_worker(rank, world, port, bits, q):
    """One rank of ColumnParallelFFN.forward: a separate process with its own
    CUDA context on cuda:0, gloo for the all-gathers (the NCCL path needs one
    GPU per rank); the layer is rebuilt from the same seeds in every process."""
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        hidden, heads, ffn, T = 256, 4, 1024, 300
        p = synth.layer_params(hidden, heads, ffn, 0)
        scales = dict(s_qkv_in=0.55, s_o_in=0.2, s_ffn1_in=0.56, s_ffn2_in=0.031 if bits == 4 else 0.0021)
        L = model.build_layer(p, bits, DEV, scales)
        h1 = torch.from_numpy(synth.activations(T, hidden, seed=4)).to(DEV)
        lo, hi = model.act_range(bits)
        codes = M.mkq_quantize_pack(h1, torch.tensor([L.scales["s_ffn1_in"]], device=DEV), bits, lo, hi)
        out = D.ColumnParallelFFN(L, rank, world).forward(codes, h1)
        torch.cuda.synchronize()
        ok = None
        if rank == 0:   # the single-process FFN + LN2 on the same inputs
            gemm = M.mkq_gemm_w4a4 if bits == 4 else M.mkq_gemm_w8a8
            t = L.t
            a2 = gemm(codes, t["w_1"], L.scales["s_ffn1_in"], t["sw_1"], t["b_1"],
                      mode=M.OUT_I4 if bits == 4 else M.OUT_I8, gelu=True, s_out=L.scales["s_ffn2_in"], qmin=lo,
                      qmax=hi, K=hidden)
            f = gemm(a2, t["w_2"], L.scales["s_ffn2_in"], t["sw_2"], t["b_2"], mode=M.OUT_F32, K=ffn)
            ref = M.mkq_residual_layernorm(f, h1, t["ln2_g"], t["ln2_b"], L.ln_eps)
            ok = bool(torch.equal(out, ref))
        q.put((rank, ok, bool(torch.isfinite(out).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bits", [4, 8])
def test_column_parallel_forward_two_processes(bits):
    """ColumnParallelFFN.forward end to end in 2 processes (gloo all-gathers)
    equals the single-GPU FFN + LN2 bit for bit."""
    import socket
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = [ctx.Process(target=_cp_worker, args=(r, world, port, bits, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0][1] is True
    assert all(r[2] for r in res)
