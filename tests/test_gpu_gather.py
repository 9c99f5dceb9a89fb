"""NEXT(4) fused all-gather: the FFN1 GEMM epilogue stores
each rank's int4 column block into every rank's gathered FFN2-input buffer
(mkq_gemm_w4a4_gather) and signals per-buffer arrival counters.

Checked against the oracle (Eq.1 + GELU + requant, bit-exact codes), against
the unfused GEMM + interleave, for the counter protocol, and end to end in
two processes that map each other's buffers through CUDA IPC."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

from paper_2203_13483_b200 import dist as D  # noqa: E402
from paper_2203_13483_b200 import mkq as M  # noqa: E402
from paper_2203_13483_b200 import model  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _problem(T, K, F, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(-8, 8, (T, K)).astype(np.int8)
    W = rng.integers(-7, 8, (F, K)).astype(np.int8)
    s_w = rng.uniform(1e-3, 5e-3, F).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, F).astype(np.float32)
    return A, W, s_w, b


def _simulate(A, W, s_w, b, world, s_a, s_out, reps=1):
    """Every simulated rank r launches its block's GEMM into all `world`
    buffers (all local here); returns (buffers, counters, arrivals)."""
    T, K = A.shape
    F = W.shape[0]
    Fl = F // world
    a = dev(oracle.pack_int4(A))
    bufs = [torch.full((T, F // 2), 0xAA, dtype=torch.uint8, device=DEV) for _ in range(world)]
    cnt = torch.zeros((world, 64), dtype=torch.int32, device=DEV)
    tab = M.mkq_requant_table(True, float(s_out), -8, 7, DEV)
    for _ in range(reps):
        for r in range(world):
            w = dev(oracle.pack_int4(W[r * Fl:(r + 1) * Fl]))
            M.mkq_gemm_w4a4_gather(a, w, float(s_a), dev(s_w[r * Fl:(r + 1) * Fl]), dev(b[r * Fl:(r + 1) * Fl]),
                                   [t.data_ptr() for t in bufs], [cnt[g].data_ptr() for g in range(world)],
                                   col0=r * Fl, ldo=F // 2, s_out=float(s_out), K=K, requant_table=tab)
    return bufs, cnt, M.mkq_gemm_gather_arrivals(T, Fl)


@pytest.mark.parametrize("T,K,F,world", [(300, 256, 1024, 2), (300, 256, 1024, 4), (1, 64, 512, 2),
                                         (513, 1024, 2048, 8), (4096 + 77, 1024, 4096, 4)])
def test_gather_codes_match_oracle(T, K, F, world):
    A, W, s_w, b = _problem(T, K, F, T + F)
    s_a, s_out = np.float32(0.31), np.float32(0.05)
    bufs, cnt, arr = _simulate(A, W, s_w, b, world, s_a, s_out)
    torch.cuda.synchronize()
    rows = np.arange(T) if T <= 1024 else np.r_[0:64, T - 77:T]   # sampled rows at the large size
    ref = oracle.pack_int4(oracle.linear(A[rows], W, s_a, s_w, b, mode=oracle.OUT_I4, gelu=True, s_out=s_out,
                                         qmin_out=-8, qmax_out=7))
    for g in range(world):
        assert np.array_equal(bufs[g].cpu().numpy()[rows], ref), f"buffer {g}"
    # every buffer's counter saw one increment per CTA of every rank's launch
    assert arr > 0
    assert cnt[:, 0].tolist() == [world * arr] * world
    assert not cnt[:, 1:].any()


def test_gather_equals_unfused_gemm_and_interleave():
    """Same codes as mkq_gemm_w4a4 per rank + the NCCL-path reassembly."""
    T, K, F, world = 2048 + 5, 1024, 4096, 2
    A, W, s_w, b = _problem(T, K, F, 9)
    s_a, s_out = np.float32(0.27), np.float32(0.043)
    bufs, _, _ = _simulate(A, W, s_w, b, world, s_a, s_out)
    full = M.mkq_gemm_w4a4(dev(oracle.pack_int4(A)), dev(oracle.pack_int4(W)), float(s_a), dev(s_w), dev(b),
                           mode=M.OUT_I4, gelu=True, s_out=float(s_out), K=K)
    for g in range(world):
        assert torch.equal(bufs[g], full)


def test_gather_counters_accumulate_over_calls():
    T, K, F, world = 300, 256, 1024, 2
    A, W, s_w, b = _problem(T, K, F, 3)
    _, cnt, arr = _simulate(A, W, s_w, b, world, np.float32(0.3), np.float32(0.05), reps=3)
    torch.cuda.synchronize()
    assert cnt[:, 0].tolist() == [3 * world * arr] * world
    # the consumer-side wait returns once the target is reached
    M.mkq_wait_counter(cnt[0].data_ptr(), 3 * world * arr)
    torch.cuda.synchronize()


_WAIT_PROG = r"""
import torch
from paper_2203_13483_b200 import mkq as M
c = torch.zeros(64, dtype=torch.int32, device="cuda")
out = torch.zeros(1, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
# load every kernel first: with lazy module loading, loading a kernel while
# another one spins on the device waits for it (a self-inflicted deadlock)
M.mkq_wait_counter(c.data_ptr(), 0)
out.add_(c[0]); torch.cuda._sleep(1000); c[0] = 5; c.zero_(); out.zero_()
torch.cuda.synchronize()
with torch.cuda.stream(s1):
    M.mkq_wait_counter(c.data_ptr(), 5, stream=s1)
    out.add_(c[0])       # runs after the wait: sees 5
with torch.cuda.stream(s2):
    torch.cuda._sleep(2_000_000)
    c[0] = 5
torch.cuda.synchronize()
assert int(out.item()) == 5, int(out.item())
print("ok")
"""


def test_wait_counter_blocks_stream_until_signalled():
    """A wait on stream s1 holds back s1's later work until stream s2 writes
    the counter (own process, bounded: a hang fails instead of blocking)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _WAIT_PROG], cwd=root, capture_output=True, text=True, timeout=180)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_gather_validation():
    a = torch.zeros((16, 128), dtype=torch.uint8, device=DEV)
    w = torch.zeros((256, 128), dtype=torch.uint8, device=DEV)
    s_w = torch.ones(256, device=DEV)
    buf = torch.zeros((16, 256), dtype=torch.uint8, device=DEV)
    c = torch.zeros(64, dtype=torch.int32, device=DEV)
    ok = dict(col0=0, ldo=256, s_out=0.05)
    M.mkq_gemm_w4a4_gather(a, w, 0.3, s_w, None, [buf.data_ptr()], [c.data_ptr()], **ok)
    with pytest.raises(RuntimeError):   # no buffers / too many
        M.mkq_gemm_w4a4_gather(a, w, 0.3, s_w, None, [], [], **ok)
    with pytest.raises(RuntimeError):
        M.mkq_gemm_w4a4_gather(a, w, 0.3, s_w, None, [buf.data_ptr()] * 9, [c.data_ptr()] * 9, **ok)
    with pytest.raises(RuntimeError):   # N % 256
        M.mkq_gemm_w4a4_gather(a, w[:128], 0.3, s_w, None, [buf.data_ptr()], [c.data_ptr()], **ok)
    with pytest.raises(RuntimeError):   # block past the row
        M.mkq_gemm_w4a4_gather(a, w, 0.3, s_w, None, [buf.data_ptr()], [c.data_ptr()], col0=544, ldo=256,
                               s_out=0.05)
    with pytest.raises(RuntimeError):   # K > 1024 (the FFN1 shape only)
        a2 = torch.zeros((16, 1024), dtype=torch.uint8, device=DEV)
        w2 = torch.zeros((256, 1024), dtype=torch.uint8, device=DEV)
        M.mkq_gemm_w4a4_gather(a2, w2, 0.3, s_w, None, [buf.data_ptr()], [c.data_ptr()], **ok)
    torch.cuda.synchronize()


def test_column_parallel_fused_single_process():
    """ColumnParallelFFN.forward_fused at world 1 (its own buffer only)
    equals forward()."""
    hidden, heads, ffn, T = 256, 4, 1024, 300
    p = synth.layer_params(hidden, heads, ffn, 0)
    L = model.build_layer(p, 4, DEV, dict(s_qkv_in=0.55, s_o_in=0.2, s_ffn1_in=0.56, s_ffn2_in=0.031))
    h1 = torch.from_numpy(synth.activations(T, hidden, seed=4)).to(DEV)
    codes = M.mkq_quantize_pack(h1, torch.tensor([L.scales["s_ffn1_in"]], device=DEV), 4, -8, 7)
    cp = D.ColumnParallelFFN(L, 0, 1)
    ref = cp.forward(codes, h1, gather=lambda x: x[None])
    cp.setup_fused_gather(T)
    for _ in range(2):
        out = cp.forward_fused(codes, h1, gather=lambda x: x[None])
        assert torch.equal(out, ref)
    cp.close_fused_gather()


def _fused_worker(rank, world, port, q):
    """One rank of forward_fused in its own process on cuda:0: the peers'
    gathered buffers and counters are CUDA-IPC mappings; gloo carries the
    handle exchange and the (unfused) second all-gather."""
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        hidden, heads, ffn, T = 256, 4, 1024, 300
        p = synth.layer_params(hidden, heads, ffn, 0)
        L = model.build_layer(p, 4, DEV, dict(s_qkv_in=0.55, s_o_in=0.2, s_ffn1_in=0.56, s_ffn2_in=0.031))
        h1 = torch.from_numpy(synth.activations(T, hidden, seed=4)).to(DEV)
        codes = M.mkq_quantize_pack(h1, torch.tensor([L.scales["s_ffn1_in"]], device=DEV), 4, -8, 7)
        cp = D.ColumnParallelFFN(L, rank, world)
        cp.setup_fused_gather(T)
        dist.barrier()
        outs = [cp.forward_fused(codes, h1) for _ in range(3)]
        torch.cuda.synchronize()
        dist.barrier()
        ok = None
        if rank == 0:
            t = L.t
            a2 = M.mkq_gemm_w4a4(codes, t["w_1"], L.scales["s_ffn1_in"], t["sw_1"], t["b_1"], mode=M.OUT_I4,
                                 gelu=True, s_out=L.scales["s_ffn2_in"], K=hidden)
            f = M.mkq_gemm_w4a4(a2, t["w_2"], L.scales["s_ffn2_in"], t["sw_2"], t["b_2"], mode=M.OUT_F32, K=ffn)
            ref = M.mkq_residual_layernorm(f, h1, t["ln2_g"], t["ln2_b"], L.ln_eps)
            ok = all(bool(torch.equal(o, ref)) for o in outs) and bool(torch.equal(cp.gbuf, a2))
        cnt = int(cp.counter[0].item())
        q.put((rank, ok, cnt == 3 * world * cp.arrivals))
        cp.close_fused_gather()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_column_parallel_fused_two_processes_ipc():
    """forward_fused in 2 processes sharing buffers through CUDA IPC equals
    the single-GPU FFN + LN2 bit for bit, three calls in a row."""
    import socket
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0][1] is True
    assert all(r[2] for r in res)
