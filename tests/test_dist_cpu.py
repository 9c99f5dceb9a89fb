"""Multi-process host logic of the multi-GPU paths on CPU (gloo, world 2):
row / varlen sharding, the rank-major all-gather + interleave, max over
ranks, and the column-parallel FFN decomposition (per-rank column blocks
computed with the oracle) reproducing the single-process FFN bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import layer as OL
import synth
from paper_2203_13483_b200 import dist as D


def test_row_shard_covers_and_balances():
    for n in [1, 7, 32, 256, 1000]:
        for w in [1, 2, 3, 4, 8]:
            parts = [D.row_shard(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_varlen_shard_contiguous_and_balanced():
    L = synth.varlen_seqlens(64, 2298, 128, seed=3)
    for w in [1, 2, 4, 8]:
        parts = [D.varlen_shard(L, w, r) for r in range(w)]
        assert parts[0][0] == 0 and parts[-1][1] == len(L)
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
        toks = [sum(L[a:b]) for a, b in parts]
        assert sum(toks) == sum(L)
        assert max(toks) - min(toks) <= 2 * max(L)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # all-gather + interleave ordering
        blk = torch.arange(6 * 4, dtype=torch.int32).reshape(6, 4) + 1000 * rank
        g = D.gather_blocks(blk, world)
        full = D.interleave_reference(g)
        ok_gather = bool(torch.equal(full[:, 4 * rank:4 * rank + 4], blk))
        mx = D.max_over_ranks(float(rank * 3 + 1))
        # column-parallel FFN: per-rank column blocks with the oracle
        h, F, bits = 64, 256, 4
        p = synth.layer_params(h, 2, F, 0)
        w1 = OL.prepare_weight(p.w_1, p.b_1, bits)
        w2 = OL.prepare_weight(p.w_2, p.b_2, bits)
        x = synth.activations(16, h, seed=9)
        s_in, s_mid = np.float32(0.55), np.float32(0.35)
        codes = oracle.quantize(x, s_in, -8, 7)
        Fl, hl = F // world, h // world
        a_loc = oracle.linear(codes, w1.codes[rank * Fl:(rank + 1) * Fl], s_in, w1.s_w[rank * Fl:(rank + 1) * Fl],
                              w1.bias[rank * Fl:(rank + 1) * Fl], mode=oracle.OUT_I4, gelu=True, s_out=s_mid)
        a_packed = torch.from_numpy(oracle.pack_int4(a_loc))
        a_full = D.interleave_reference(D.gather_blocks(a_packed, world)).numpy()
        a_codes = oracle.unpack_int4(a_full, F)
        f_loc = oracle.linear(a_codes, w2.codes[rank * hl:(rank + 1) * hl], s_mid, w2.s_w[rank * hl:(rank + 1) * hl],
                              w2.bias[rank * hl:(rank + 1) * hl])
        f_full = D.interleave_reference(D.gather_blocks(torch.from_numpy(f_loc), world)).numpy()
        a_ref = oracle.linear(codes, w1.codes, s_in, w1.s_w, w1.bias, mode=oracle.OUT_I4, gelu=True, s_out=s_mid)
        f_ref = oracle.linear(a_ref, w2.codes, s_mid, w2.s_w, w2.bias)
        q.put((rank, ok_gather, mx, bool(np.array_equal(a_codes, a_ref)),
               bool(np.array_equal(f_full.view(np.uint32), f_ref.view(np.uint32)))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_column_parallel_ffn():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok_gather, mx, ok_a, ok_f in res:
        assert ok_gather, rank
        assert mx == 4.0
        assert ok_a and ok_f, rank
