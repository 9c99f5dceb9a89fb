"""Multi-GPU plumbing for the W4A4 BERT layer.

* Row sharding (the scaling headline): every hot-path step is independent
  per token row and attention needs whole sequences, so ranks take disjoint
  sets of whole sequences; weights are replicated; no collective on the data
  path ("scaling": "weak" in bench.py).
* Column-parallel FFN (the NCCL variant): rank r holds W^1 rows
  [r F/g, (r+1) F/g) and W^2 rows [r h/g, (r+1) h/g).  FFN1 (GELU + requant
  fused) produces the rank's int4 column block of the FFN2 input; an
  all_gather of the packed codes over NCCL plus `mkq_interleave_blocks`
  rebuilds the [T, F/2] code matrix (column order = W^2's K order, so no
  permutation of W^2 is needed); FFN2 produces the rank's fp32 output
  columns; a second all_gather + interleave rebuilds [T, h] for LN2.  Every
  output element is computed by exactly the kernel arithmetic of the
  single-GPU layer, so the result is bit-identical to it.

torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used for process
groups and the all-gathers only; all arithmetic runs in libmkq kernels.
"""
from __future__ import annotations

import os
from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def init_from_env(backend: str = "nccl") -> Tuple[int, int, int]:
    """Initialise the default process group from torchrun's environment;
    returns (rank, world, local_rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return rank, world, local


def row_shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split of n units (sequences): [start, stop)."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def varlen_shard(seqlens: Sequence[int], world: int, rank: int) -> Tuple[int, int]:
    """Contiguous split of variable-length sequences balancing token counts
    (greedy prefix cut at multiples of total/world): [first, last) sequence."""
    total = sum(seqlens)
    cuts = [0]
    acc = 0
    target = 1
    for i, L in enumerate(seqlens):
        acc += L
        while target < world and acc >= target * total / world:
            cuts.append(i + 1)
            target += 1
    while len(cuts) < world:
        cuts.append(len(seqlens))
    cuts.append(len(seqlens))
    return cuts[rank], cuts[rank + 1]


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_blocks(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """all_gather of a [rows, cb] block per rank -> [world, rows, cb] (rank-major)."""
    out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    elif local.is_cuda:   # gloo with device tensors (the multi-process tests on one GPU): staged via host
        host = torch.empty((world,) + tuple(local.shape), dtype=local.dtype)
        dist.all_gather(list(host.unbind(0)), local.contiguous().cpu(), group=group)
        out.copy_(host)
    else:   # gloo (CPU tests): list form
        dist.all_gather(list(out.unbind(0)), local.contiguous(), group=group)
    return out


def interleave_reference(blocks: torch.Tensor) -> torch.Tensor:
    """[g, rows, c] -> [rows, g*c]: the host-side definition of the
    reassembly (used by the CPU tests; the GPU path uses mkq_interleave_blocks)."""
    g, rows, c = blocks.shape
    return blocks.permute(1, 0, 2).reshape(rows, g * c)


class ColumnParallelFFN:
    """The FFN block of one quantized layer, split by output columns."""

    def __init__(self, layer, rank: int, world: int):
        from . import mkq as M
        self.M = M
        self.layer, self.rank, self.world = layer, rank, world
        h, F, bits = layer.hidden, layer.ffn, layer.bits
        assert F % (32 * world) == 0 and h % (32 * world) == 0, "column blocks must be multiples of 32"
        self.Fl, self.hl = F // world, h // world
        t = layer.t
        f0, f1 = rank * self.Fl, (rank + 1) * self.Fl
        o0, o1 = rank * self.hl, (rank + 1) * self.hl
        self.w1, self.sw1, self.b1 = t["w_1"][f0:f1].contiguous(), t["sw_1"][f0:f1].contiguous(), t["b_1"][f0:f1].contiguous()
        self.w2, self.sw2, self.b2 = t["w_2"][o0:o1].contiguous(), t["sw_2"][o0:o1].contiguous(), t["b_2"][o0:o1].contiguous()
        self.lo, self.hi = (-8, 7) if bits == 4 else (-128, 127)
        self.gemm = M.mkq_gemm_w4a4 if bits == 4 else M.mkq_gemm_w8a8

    def ffn1_local(self, codes_h1: torch.Tensor, stream=None) -> torch.Tensor:
        L, M = self.layer, self.M
        mode = M.OUT_I4 if L.bits == 4 else M.OUT_I8
        return self.gemm(codes_h1, self.w1, L.scales["s_ffn1_in"], self.sw1, self.b1, mode=mode, gelu=True,
                         s_out=L.scales["s_ffn2_in"], qmin=self.lo, qmax=self.hi, K=L.hidden, stream=stream,
                         requant_table=L.table if L.table is not None else True)

    def ffn2_local(self, a2_full: torch.Tensor, stream=None) -> torch.Tensor:
        L, M = self.layer, self.M
        return self.gemm(a2_full, self.w2, L.scales["s_ffn2_in"], self.sw2, self.b2, mode=M.OUT_F32, K=L.ffn,
                         stream=stream)

    # ---------------------------------------------------------------- NEXT(4) fused all-gather
    def setup_fused_gather(self, T: int, group=None) -> None:
        """Allocate this rank's gathered FFN2-input buffer [T, F/2] (packed
        int4) and its arrival counter, exchange CUDA-IPC handles with the
        other ranks (dist.all_gather_object) and map theirs.  After this,
        forward_fused writes every rank's FFN1 column block straight into
        every rank's buffer from the GEMM epilogue (mkq_gemm_w4a4_gather):
        no NCCL call and no interleave for the first all-gather."""
        M, L = self.M, self.layer
        if L.bits != 4 or self.Fl % 256 or L.hidden > 1024:
            raise ValueError("fused all-gather: W4A4 layers with F/world % 256 == 0 and hidden <= 1024")
        dev = L.t["w_1"].device
        self.T_fused = T
        self.gbuf = torch.zeros((T, L.ffn // 2), dtype=torch.uint8, device=dev)
        self.counter = torch.zeros(64, dtype=torch.int32, device=dev)   # [0] used; 256-byte slot
        self.arrivals = M.mkq_gemm_gather_arrivals(T, self.Fl)
        self.epoch = 0
        mine = (M.mkq_ipc_get_handle(self.gbuf), M.mkq_ipc_get_handle(self.counter))
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self._mapped = []
        outs, cnts = [], []
        for r, ((hb, ob), (hc, oc)) in enumerate(allh):
            if r == self.rank:
                outs.append(self.gbuf.data_ptr())
                cnts.append(self.counter.data_ptr())
                continue
            bb, bc = M.mkq_ipc_open_handle(hb), M.mkq_ipc_open_handle(hc)
            self._mapped += [bb, bc]
            outs.append(bb + ob)
            cnts.append(bc + oc)
        self.outs, self.cnts = outs, cnts

    def close_fused_gather(self) -> None:
        for b in getattr(self, "_mapped", []):
            self.M.mkq_ipc_close(b)
        self._mapped = []

    def forward_fused(self, codes_h1: torch.Tensor, h1: torch.Tensor,
                      gather: Optional[Callable[[torch.Tensor], torch.Tensor]] = None, stream=None) -> torch.Tensor:
        """forward() with the FFN1 all-gather fused into the FFN1 GEMM.  The
        caller's ranks must all call it (the counters count every rank's
        CTAs).  Reuse of the gathered buffers across calls is ordered by the
        second all-gather: a rank can only pass it once every rank's FFN2
        (the reader of its buffer) has run."""
        M, L = self.M, self.layer
        gather = gather or (lambda x: gather_blocks(x, self.world))
        T = h1.shape[0]
        assert T == self.T_fused, "setup_fused_gather(T) for this token count"
        self.epoch += 1
        M.mkq_gemm_w4a4_gather(codes_h1, self.w1, L.scales["s_ffn1_in"], self.sw1, self.b1, self.outs, self.cnts,
                               col0=self.rank * self.Fl, ldo=L.ffn // 2, s_out=L.scales["s_ffn2_in"], gelu=True,
                               qmin=self.lo, qmax=self.hi, K=L.hidden,
                               requant_table=L.table if L.table is not None else None, stream=stream)
        M.mkq_wait_counter(self.counter.data_ptr(), self.epoch * self.world * self.arrivals, stream=stream)
        f_loc = self.ffn2_local(self.gbuf, stream)                   # [T, hl] fp32
        f_blocks = gather(f_loc)                                     # [g, T, hl]
        f = M.mkq_interleave_blocks(f_blocks.view(torch.uint8), self.world, T, self.hl * 4,
                                    stream=stream).view(torch.float32)
        return M.mkq_residual_layernorm(f, h1, L.t["ln2_g"], L.t["ln2_b"], L.ln_eps, stream=stream)

    def forward(self, codes_h1: torch.Tensor, h1: torch.Tensor,
                gather: Optional[Callable[[torch.Tensor], torch.Tensor]] = None, stream=None) -> torch.Tensor:
        """codes_h1 [T, K-codes] and h1 [T, h] fp32 on every rank -> h_out [T, h]."""
        M, L = self.M, self.layer
        gather = gather or (lambda x: gather_blocks(x, self.world))
        T = h1.shape[0]
        a2_loc = self.ffn1_local(codes_h1, stream)
        a2_blocks = gather(a2_loc)                                   # [g, T, Fl bytes]
        a2 = M.mkq_interleave_blocks(a2_blocks, self.world, T, a2_loc.shape[1], stream=stream)
        if L.bits == 8:
            a2 = a2.view(torch.int8)
        f_loc = self.ffn2_local(a2, stream)                          # [T, hl] fp32
        f_blocks = gather(f_loc)                                     # [g, T, hl]
        f = M.mkq_interleave_blocks(f_blocks.view(torch.uint8), self.world, T, self.hl * 4,
                                    stream=stream).view(torch.float32)
        return M.mkq_residual_layernorm(f, h1, L.t["ln2_g"], L.t["ln2_b"], L.ln_eps, stream=stream)
