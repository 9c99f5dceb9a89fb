#!/usr/bin/env python3
"""bench.py -- BERT int4 (W4A4) layer throughput on B200, 1..8 GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1: launched by torchrun, one rank per GPU, NCCL for barrier/timing)

Workload (BASELINE.json configs[3], at N=1 exactly that config per rank):
one BERT-large post-LN encoder layer (hidden 1024, 16 heads, FFN 4096),
W4A4 on all six weight GEMMs, batch 256 x seq 512 = 131072 tokens per rank,
synthetic seeded data and random-init weights (synth/).  Scaling is weak:
every rank runs its own batch of whole sequences (row sharding, no
data-path collective).

A step is one pass of the whole hot path (§8a rows a1-a8) over one batch:
mkq_bert_layer = quantize -> QKV GEMM (fp16 out) -> attention (+fused
quantize) -> W^A GEMM -> residual+LN (+fused quantize) -> FFN1 GEMM (GELU +
requant fused) -> FFN2 GEMM -> residual+LN.

metric / value: "W4A4 GEMM TOPS" = the layer's linear-GEMM integer ops
(2*tokens*(3h^2 + h^2 + 2*h*ffn), the BASELINE.md 'effective int4 layer
throughput' methodology) / layer time, summed over ranks.  Layer latency,
per-stage times, the dominant kernel's roofline and the paper-style fp32 /
bf16 layer comparison are reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CFG = dict(batch=256, seq=512, hidden=1024, heads=16, ffn=4096, bits=4)
WORKLOAD = "bert_large_w4a4_layer_b256_s512 (BASELINE.json configs[3], per rank)"


def linear_ops(tokens, hidden, ffn):
    return 2.0 * tokens * (3 * hidden * hidden + hidden * hidden + 2 * hidden * ffn)


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        src = "measured"
    except Exception:
        src = "fallback"
    hbm = float(p.get("hbm_gbs", 6650.0))
    bf16_burst = float(p.get("bf16_tflops", 1590.0))
    bf16_sus = float(p.get("bf16_tflops_sustained", 1400.0))
    # int8 dense = 2x bf16 dense (nominal 4.5 / 2.25 PFLOP/s; B200_PROFILING.md)
    return dict(src=src, hbm_gbs=hbm, int8_tops_burst=2 * bf16_burst, int8_tops_sustained=2 * bf16_sus,
                bf16_tflops=bf16_burst, bf16_tflops_sustained=bf16_sus)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock / power / throttle reasons sampled DURING the timed region:
    NVML (pynvml) every 10 ms in a thread, nvidia-smi as the fallback."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []          # (sm_mhz, max_mhz, power_w, set(reasons))
        self._stop = threading.Event()
        self._t = None
        self.src = None

    def _nvml(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        self.src = "nvml"
        while not self._stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((float(sm), float(mx), pw, {k for k, b in bits.items() if r & b}))
            self._stop.wait(0.01)

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.src = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                c = [x.strip() for x in out.split(",")]
                if len(c) >= 7:
                    self.rows.append((float(c[0]), float(c[1]), float(c[2]),
                                      {self.NAMES[i] for i in range(4) if c[3 + i] == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.1)

    def _run(self):
        try:
            self._nvml()
        except Exception:
            self._smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_mhz_min": min(sm), "power_w_max": round(max(r[2] for r in self.rows), 1),
                "reasons": sorted(set().union(*[r[3] for r in self.rows])), "samples": len(self.rows),
                "source": self.src}


def peak_regime(clk):
    """'burst' if the timed region ran at (nearly) max SM clock with no power
    cap, else 'sustained' (B200_PROFILING.md: the burst figure for a kernel
    timed alone, the sustained one under the power cap)."""
    sm, mx = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    if sm and mx and sm >= 0.95 * mx and "sw_power_cap" not in clk.get("reasons", []):
        return "burst"
    return "sustained"


# ------------------------------------------------------------------ our arm
def setup_layer(torch, dev, rank):
    import synth
    from paper_2203_13483_b200 import model
    p = synth.layer_params(CFG["hidden"], CFG["heads"], CFG["ffn"], layer=0)
    L = model.build_layer(p, CFG["bits"], dev)
    # offline calibration on a 4-sequence calibration batch
    ncal = 4
    hc = torch.from_numpy(synth.hidden_states(ncal, CFG["seq"], CFG["hidden"], seed=1000000)).to(dev)
    model.calibrate(L, hc, ncal, CFG["seq"])
    return L, p


def stage_calls(M, L, h_in, B, T, stream):
    """The launches of mkq_bert_layer as separate C-ABI calls (same kernels,
    same arguments) so each can be bracketed by CUDA events: eight stages, or
    six when the layer fuses residual + LayerNorm into the W^A and W^2 GEMMs
    (mkq_gemm_residual_ln, NEXT(4); L.fused_ln(T))."""
    import torch
    hd, F, bits = L.hidden, L.ffn, L.bits
    t = L.t
    s = L.scales
    buf = {}
    dev = h_in.device
    buf["c_in"] = torch.empty((T, hd // 2), dtype=torch.uint8, device=dev)
    buf["qkv"] = torch.empty((T, 3 * hd), dtype=torch.float16, device=dev)
    buf["c_oa"] = torch.empty((T, hd // 2), dtype=torch.uint8, device=dev)
    buf["o"] = torch.empty((T, hd), dtype=torch.float32, device=dev)
    buf["h1"] = torch.empty((T, hd), dtype=torch.float32, device=dev)
    buf["c_h1"] = torch.empty((T, hd // 2), dtype=torch.uint8, device=dev)
    buf["a2"] = torch.empty((T, F // 2), dtype=torch.uint8, device=dev)
    buf["f"] = torch.empty((T, hd), dtype=torch.float32, device=dev)
    buf["out"] = torch.empty((T, hd), dtype=torch.float32, device=dev)
    sq = torch.tensor([s["s_qkv_in"]], device=dev)
    S = CFG["seq"]
    calls = [
        ("quantize_in", lambda: M.mkq_quantize_pack(h_in, sq, 4, -8, 7, out=buf["c_in"], stream=stream), 0),
        ("gemm_qkv", lambda: M.mkq_gemm_w4a4(buf["c_in"], t["w_qkv"], s["s_qkv_in"], t["sw_qkv"], t["b_qkv"],
                                             mode=M.OUT_F16, out=buf["qkv"], K=hd, stream=stream), 2.0 * T * 3 * hd * hd),
        ("attention", lambda: M.mkq_attention(buf["qkv"], L.heads, B, S, None, mode=M.OUT_I4, s_out=s["s_o_in"],
                                              out=buf["c_oa"], stream=stream), 4.0 * T * S * hd),
        ("gemm_o", lambda: M.mkq_gemm_w4a4(buf["c_oa"], t["w_o"], s["s_o_in"], t["sw_o"], t["b_o"], mode=M.OUT_F32,
                                           out=buf["o"], K=hd, stream=stream), 2.0 * T * hd * hd),
        ("ln1_quant", lambda: M.mkq_residual_layernorm(buf["o"], h_in, t["ln1_g"], t["ln1_b"], L.ln_eps, bits=4,
                                                       s_q=s["s_ffn1_in"], y=buf["h1"], q=buf["c_h1"], stream=stream), 0),
        ("gemm_ffn1", lambda: M.mkq_gemm_w4a4(buf["c_h1"], t["w_1"], s["s_ffn1_in"], t["sw_1"], t["b_1"],
                                              mode=M.OUT_I4, gelu=True, s_out=s["s_ffn2_in"], out=buf["a2"], K=hd,
                                              stream=stream, requant_table=L.table), 2.0 * T * hd * F),
        ("gemm_ffn2", lambda: M.mkq_gemm_w4a4(buf["a2"], t["w_2"], s["s_ffn2_in"], t["sw_2"], t["b_2"],
                                              mode=M.OUT_F32, out=buf["f"], K=F, stream=stream), 2.0 * T * hd * F),
        ("ln2", lambda: M.mkq_residual_layernorm(buf["f"], buf["h1"], t["ln2_g"], t["ln2_b"], L.ln_eps,
                                                 y=buf["out"], stream=stream), 0),
    ]
    if L.fused_ln(T):
        fused = {
            "gemm_o_ln1": (lambda: M.mkq_gemm_residual_ln(
                buf["c_oa"], t["w_o"], s["s_o_in"], t["sw_o"], t["b_o"], h_in, t["ln1_g"], t["ln1_b"], L.ln_eps, K=hd,
                q_bits=4, s_q=s["s_ffn1_in"], y=buf["h1"], q=buf["c_h1"], stream=stream), 2.0 * T * hd * hd),
            "gemm_ffn2_ln2": (lambda: M.mkq_gemm_residual_ln(
                buf["a2"], t["w_2"], s["s_ffn2_in"], t["sw_2"], t["b_2"], buf["h1"], t["ln2_g"], t["ln2_b"], L.ln_eps,
                K=F, y=buf["out"], stream=stream), 2.0 * T * hd * F),
        }
        calls = [c for c in calls if c[0] not in ("gemm_o", "ln1_quant", "gemm_ffn2", "ln2")]
        calls.insert(3, ("gemm_o_ln1",) + fused["gemm_o_ln1"])
        calls.append(("gemm_ffn2_ln2",) + fused["gemm_ffn2_ln2"])
    return calls, buf


def load_traffic():
    """Per-launch DRAM bytes of each stage from the newest committed ncu
    --set full summary (tools/summarize_ncu.py -> profiles/r*_layer_traffic.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_layer_traffic.json")))
    if not files:
        return {}, None
    try:
        return json.load(open(files[-1])), os.path.relpath(files[-1], ROOT)
    except Exception:
        return {}, None


def stage_bytes(T, hd, F):
    """Algorithmic HBM bytes per launch."""
    return {
        "quantize_in": T * hd * 4.5,
        "gemm_qkv": T * hd / 2 + 3 * hd * hd / 2 + T * 3 * hd * 2,
        "attention": T * 3 * hd * 2 + T * hd / 2,
        "gemm_o": T * hd / 2 + hd * hd / 2 + T * hd * 4,
        "ln1_quant": T * hd * (4 + 4 + 4 + 0.5),
        "gemm_ffn1": T * hd / 2 + F * hd / 2 + T * F / 2,
        "gemm_ffn2": T * F / 2 + F * hd / 2 + T * hd * 4,
        "ln2": T * hd * 12,
        # fused residual + LN (NEXT(4)): codes + weights + residual in, y (+ codes) out
        "gemm_o_ln1": T * hd / 2 + hd * hd / 2 + T * hd * 4 + T * hd * 4 + T * hd / 2,
        "gemm_ffn2_ln2": T * F / 2 + F * hd / 2 + T * hd * 4 + T * hd * 4,
    }


def event_time(torch, fn, stream, reps, warm=2):
    """Mean device time (ms) of fn() over reps back-to-back calls on stream."""
    with torch.cuda.stream(stream):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def graph_time(torch, fn, dev, reps=100, inner=1):
    """Device time (ms) per fn() call: `inner` calls captured in one CUDA graph,
    replayed reps // inner times (the paper's mean of 100 rounds)."""
    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        for _ in range(3):
            fn(st)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(inner):
                fn(st)
        g.replay()
        torch.cuda.synchronize(dev)
        n = max(1, reps // inner)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(n):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / (n * inner)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2203_13483_b200 import dist as D
    from paper_2203_13483_b200 import mkq as M

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import synth

    L, p = setup_layer(torch, dev, rank)
    S, hd, F = CFG["seq"], CFG["hidden"], CFG["ffn"]
    B_total = CFG["batch"]
    if args.scaling == "strong":   # the BASELINE configs[3] batch, whole sequences sharded over the ranks
        b0, b1 = D.row_shard(B_total, world, rank)
        B = b1 - b0
    else:                          # every rank runs a full configs[3] batch
        b0, B = rank * B_total, B_total
    T = B * S
    h_host = synth.hidden_states(B, S, hd, seed=1 + b0)
    h_in = torch.from_numpy(h_host).to(dev)
    h_out = torch.empty_like(h_in)
    ws = torch.empty(L.workspace_size(T), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def step():
        M.mkq_bert_layer(L, h_in, B, S, None, h_out=h_out, ws=ws, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_ranks(x):
        if world == 1:
            return x
        tt = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t_max = max_ranks(ms)
    tokens_all = (B_total if args.scaling == "strong" else B_total * world) * S
    ops_all = linear_ops(tokens_all, hd, F)
    value = ops_all / (t_max * 1e-3) / 1e12
    clocks = clk.summary()
    regime = peak_regime(clocks)

    # ---- per-stage device times (same kernels, one event pair per launch; rank 0's shard)
    calls, buf = stage_calls(M, L, h_in, B, T, stream)
    nrep = max(3, min(args.steps, 10))
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in calls]
           for _ in range(nrep)]
    with torch.cuda.stream(stream):
        for c in calls:
            c[1]()
        torch.cuda.synchronize(dev)
        for r in range(nrep):
            for i, c in enumerate(calls):
                evs[r][i][0].record(stream)
                c[1]()
                evs[r][i][1].record(stream)
    torch.cuda.synchronize(dev)
    stage_ms = {c[0]: float(np.mean([evs[r][i][0].elapsed_time(evs[r][i][1]) for r in range(nrep)]))
                for i, c in enumerate(calls)}
    same = bool(torch.equal(buf["out"], h_out))
    pk = peaks()
    sb = stage_bytes(T, hd, F)
    gemms = {k: v for k, v in stage_ms.items() if k.startswith("gemm")}
    dom = max(stage_ms, key=stage_ms.get)
    ops_of = {c[0]: c[2] for c in calls}
    traffic, traffic_src = load_traffic()
    i8 = {"burst": pk["int8_tops_burst"], "sustained": pk["int8_tops_sustained"]}
    f16 = {"burst": pk["bf16_tflops"], "sustained": pk["bf16_tflops_sustained"]}

    def roofline(k):
        tr = traffic.get(k, {}).get("dram_bytes")
        base = {"kernel": k, "traffic": tr, "traffic_src": traffic_src, "algorithmic_bytes": sb[k],
                "peak_regime": regime}
        if ops_of[k] > 0:
            ach = ops_of[k] / (stage_ms[k] * 1e-3) / 1e12
            if k == "attention":   # fp16 tensor-core contraction, flops = 4*T*S*d
                pk_ = f16
                base.update(unit="TFLOP/s (fp16 dense)",
                            peak_src=f"{pk['src']} bf16_tflops{'' if regime == 'burst' else '_sustained'} "
                                     f"(fp16 = bf16 nominal rate)")
            else:                  # int8 tensor-core contraction (tcgen05 kind::i8)
                pk_ = i8
                base.update(unit="TOPS (int8 dense)",
                            peak_src=f"{pk['src']} 2 x bf16_tflops{'' if regime == 'burst' else '_sustained'} "
                                     f"(int8:bf16 nominal 4.5:2.25)")
            base.update(bound="tensor", achieved=round(ach, 1), peak=round(pk_[regime], 1),
                        frac=round(ach / pk_[regime], 4), frac_of_burst=round(ach / pk_["burst"], 4),
                        frac_of_sustained=round(ach / pk_["sustained"], 4))
            return base
        ach = sb[k] / (stage_ms[k] * 1e-3) / 1e9
        base.update(bound="hbm", achieved=round(ach, 1), peak=pk["hbm_gbs"], unit="GB/s",
                    frac=round(ach / pk["hbm_gbs"], 4), peak_src=pk["src"] + " hbm_gbs")
        return base

    roof = roofline(dom)
    roof_all = {k: {kk: v for kk, v in roofline(k).items()
                    if kk in ("bound", "achieved", "unit", "frac", "frac_of_burst", "frac_of_sustained")}
                for k in stage_ms}
    stages = {}
    for k, v in stage_ms.items():
        d = {"us": round(v * 1e3, 1), "share": round(v / sum(stage_ms.values()), 3),
             "gbs": round(sb[k] / (v * 1e-3) / 1e9, 1)}
        if ops_of[k]:
            d["tops"] = round(ops_of[k] / (v * 1e-3) / 1e12, 1)
        stages[k] = d
    gemm_ms = sum(gemms.values())
    gemm_tops = linear_ops(T, hd, F) / (gemm_ms * 1e-3) / 1e12

    # ---- e2e: host buffers through the C-ABI, H2D + layer + D2H in the timed region.
    # Whole sequences are independent, so the rank's batch is processed in chunks
    # of sequences pipelined over three streams (H2D of chunk i+1 and D2H of
    # chunk i-1 overlap the layer on chunk i); the result is bit-identical to
    # one call on the whole batch (checked below).
    h_pin = torch.from_numpy(h_host).pin_memory()
    o_pin = torch.empty(h_host.shape, dtype=torch.float32).pin_memory()
    e2e_steps = max(2, min(args.steps, 5))
    # chunks of whole sequences: more chunks shorten the un-overlapped first H2D /
    # last D2H (PCIe-bound; env MKQ_E2E_CHUNKS overrides, diagnostics)
    # (8: 12.49 ms, 16: 12.23, 32: 12.66 at C4: 2 x 537 MB at ~44 GB/s per PCIe direction)
    nch = int(os.environ.get("MKQ_E2E_CHUNKS", "0")) or next((c for c in (16, 8, 4, 2) if B % c == 0), 1)
    Bc, Tc = B // nch, (B // nch) * S
    ws_c = torch.empty(L.workspace_size(Tc), dtype=torch.uint8, device=dev)
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(nch)]
    ev_done = [torch.cuda.Event() for _ in range(nch)]

    def e2e_step():
        for c in range(nch):
            rows = slice(c * Tc, (c + 1) * Tc)
            with torch.cuda.stream(s_in):
                if c == 0:
                    s_in.wait_stream(s_out)          # previous step's D2H done before buffers are reused
                h_in[rows].copy_(h_pin[rows], non_blocking=True)
                ev_in[c].record(s_in)
            stream.wait_event(ev_in[c])
            M.mkq_bert_layer(L, h_in[rows], Bc, S, None, h_out=h_out[rows], ws=ws_c, stream=stream)
            ev_done[c].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[c])
                o_pin[rows].copy_(h_out[rows], non_blocking=True)

    e2e_step()
    barrier()
    e2e_same = bool(np.array_equal(o_pin.numpy(), buf["out"].cpu().numpy()))
    del buf
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    s_in.wait_stream(stream)
    for _ in range(e2e_steps):
        e2e_step()
    stream.wait_stream(s_out)
    e1.record(stream)
    barrier()
    e2e_ms = max_ranks(e0.elapsed_time(e1) / e2e_steps)
    del ws_c, h_pin, o_pin

    # ---- multi-GPU arms (every rank): C3 row-sharded encoder, column-parallel FFN (N > 1)
    c3_rs = c3_row_sharded(torch, dev, world, rank, barrier, max_ranks)
    colpar = None
    if world > 1:
        colpar = column_parallel_ffn(torch, L, dev, world, rank, barrier, max_ranks, stream)
    del h_out, ws

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        extras["small_configs_c1_c2"] = small_configs(torch, dev, pk, regime)
        if not args.no_compare:
            extras["paper_comparison"] = compare_float_layers(torch, p, dev, ms, args)
        if not args.no_table2:
            extras["table2_bert_base_varlen"] = table2(torch, dev)
            extras["bert_base_12l_b32s128"] = c3_encoder(torch, dev)
        extras["qat_and_calibration"] = qat_calibration(torch, M, h_in, stream, pk)

    result = None
    if rank == 0:
        cpu = None if (args.no_cpu or world > 1) else cpu_baseline(sample_seqs=1)
        result = {
            "metric": "W4A4 GEMM TOPS (effective: layer linear-GEMM int ops / BERT int4 layer time)",
            "value": round(value, 2),
            "unit": "TOPS",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(t_max, 4),
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "s4 x s4 -> s32 (int8 tcgen05), fp32 epilogue/LN, fp16 attention",
            "data": "synthetic (seeded N(0,1) activations, N(0,0.02^2) random-init BERT weights)",
            "config": {"workload": WORKLOAD, "batch_total": B_total if args.scaling == "strong" else B_total * world,
                       "batch_per_rank": B, "seq_len": S, "hidden": hd, "heads": CFG["heads"], "ffn": F, "bits": 4,
                       "tokens_per_rank": T,
                       "parallelism": f"row-shard x{world} by whole sequences ({args.scaling} scaling, no collective)",
                       "l2": "inputs > L2: 537 MB fp32 activations per full batch + ~3 GB intermediates; "
                             "weights (6.3 MB) L2-resident"},
            "layer_latency_us": round(t_max * 1e3, 1),
            "gemm_only_tops": round(gemm_tops, 1),
            "stages": stages,
            "layer_equals_staged": same,
            "roofline": roof,
            "roofline_by_stage": roof_all,
            "e2e": {"value": round(ops_all / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TOPS",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(h_host.nbytes),
                    "d2h_bytes_per_step": int(h_host.nbytes),
                    "pipeline": f"{nch} chunks of {Bc} sequences per rank over H2D / compute / D2H streams",
                    "result_equals_device_step": e2e_same},
            "gpu_launches": len(stage_ms) * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "c3_row_sharded": c3_rs,
            "column_parallel_ffn": colpar,
        }
        result.update(extras)
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def c3_row_sharded(torch, dev, world, rank, barrier, max_ranks, reps=20):
    """BASELINE.json configs[2] row-sharded: the BERT-base
    12-layer mixed-precision encoder (layers 1-6 W8A8, 7-12 W4A4)
    over the batch of 32 x 128-token sequences, 32/g whole sequences per
    rank, no collective; one CUDA graph per rank, max over ranks."""
    import synth
    from paper_2203_13483_b200 import dist as D
    from paper_2203_13483_b200 import model
    h, H, F, Btot, S = 768, 12, 3072, 32, 128
    b0, b1 = D.row_shard(Btot, world, rank)
    B = b1 - b0
    layers = []
    for i, bits in enumerate(model.bit_plan(12, 6)):
        p = synth.layer_params(h, H, F, i)
        L = model.build_layer(p, bits, dev)
        model.calibrate(L, torch.from_numpy(synth.hidden_states(4, S, h, seed=1000000 + i)).to(dev), 4, S)
        layers.append(L)
    enc = model.Encoder(layers)
    hin = torch.from_numpy(synth.hidden_states(B, S, h, seed=1 + b0)).to(dev)
    out = torch.empty_like(hin)
    barrier()
    ms = graph_time(torch, lambda st: enc(hin, B, S, out=out, stream=st), dev, reps=reps)
    t = max_ranks(ms)
    T = Btot * S
    return {"workload": "BERT-base 12 layers, 6 x W8A8 + 6 x W4A4, batch 32 x seq 128 (configs[2])",
            "n_gpus": world, "sequences_per_rank": B, "ms": round(t, 4),
            "tokens_per_s": round(T / (t * 1e-3), 1),
            "tops": round(12 * linear_ops(T, h, F) / (t * 1e-3) / 1e12, 1), "scaling": "strong",
            "timing": "CUDA graph of the 12-layer stack per rank, mean of replays, max over ranks"}


def column_parallel_ffn(torch, L, dev, world, rank, barrier, max_ranks, stream, reps=5):
    """BASELINE.json configs[3] column-parallel FFN: every rank
    holds W^1 rows [rF/g, (r+1)F/g) and W^2 rows [rh/g, (r+1)h/g) and
    processes ALL 131072 tokens; FFN1 (GELU + int4 requant fused) -> NCCL
    all_gather of the packed int4 codes -> interleave -> FFN2 -> NCCL
    all_gather of the fp32 output columns -> interleave -> residual + LN2.
    Each sub-step is timed with CUDA events on its stream; all-gather
    bandwidth is reported as NCCL's busbw against the measured 770 GB/s
    per-direction NVLink peer figure (B200_PROFILING.md)."""
    import synth
    import torch.distributed as dist
    from paper_2203_13483_b200 import dist as D
    from paper_2203_13483_b200 import mkq as M
    hd, F, S = L.hidden, L.ffn, CFG["seq"]
    T = CFG["batch"] * S
    cp = D.ColumnParallelFFN(L, rank, world)
    h1 = torch.from_numpy(synth.hidden_states(CFG["batch"], S, hd, seed=7)).to(dev)
    codes = M.mkq_quantize_pack(h1, torch.tensor([L.scales["s_ffn1_in"]], device=dev), 4, -8, 7)
    names = ("ffn1_local", "allgather_int4", "interleave_int4", "ffn2_local", "allgather_f32", "interleave_f32",
             "ln2")
    times = {n: [] for n in names}

    def once(record):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            a_loc = cp.ffn1_local(codes, stream)
            ev[1].record(stream)
            a_blk = D.gather_blocks(a_loc, world)
            ev[2].record(stream)
            a2 = M.mkq_interleave_blocks(a_blk, world, T, a_loc.shape[1], stream=stream)
            ev[3].record(stream)
            f_loc = cp.ffn2_local(a2, stream)
            ev[4].record(stream)
            f_blk = D.gather_blocks(f_loc, world)
            ev[5].record(stream)
            f = M.mkq_interleave_blocks(f_blk.view(torch.uint8), world, T, cp.hl * 4, stream=stream).view(torch.float32)
            ev[6].record(stream)
            out = M.mkq_residual_layernorm(f, h1, L.t["ln2_g"], L.t["ln2_b"], L.ln_eps, stream=stream)
            ev[7].record(stream)
        torch.cuda.synchronize(dev)
        if record:
            for i, n in enumerate(names):
                times[n].append(ev[i].elapsed_time(ev[i + 1]))
        return out

    once(False)
    barrier()
    for _ in range(reps):
        barrier()
        once(True)
    ms = {n: max_ranks(float(np.mean(v))) for n, v in times.items()}
    tot = max_ranks(float(np.sum([np.mean(v) for v in times.values()])))
    fused = None
    if os.environ.get("MKQ_BENCH_FUSED_AG") == "1":
        # NEXT(4): FFN1 with the all-gather fused into its epilogue (peer TMA
        # stores through CUDA IPC + arrival counters), then the same FFN2 path
        ref_out = once(False)
        cp.setup_fused_gather(T)
        barrier()
        out = cp.forward_fused(codes, h1, stream=stream)
        torch.cuda.synchronize(dev)
        same = bool(torch.equal(out, ref_out))
        ft = []
        for _ in range(reps):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                cp.forward_fused(codes, h1, stream=stream)
                e1.record(stream)
            torch.cuda.synchronize(dev)
            ft.append(e0.elapsed_time(e1))
        barrier()
        cp.close_fused_gather()
        same_all = max_ranks(0.0 if same else 1.0) == 0.0
        fused = {"ms_total": round(max_ranks(float(np.mean(ft))), 4), "bit_identical_to_nccl_path": same_all,
                 "collective": "FFN1 epilogue TMA stores into every rank's buffer (CUDA IPC) + counters; "
                               "NCCL all_gather for the fp32 FFN2 output"}
    g1 = T * F / 2          # bytes of the gathered int4 FFN2 input
    g2 = T * hd * 4         # bytes of the gathered fp32 FFN2 output
    busbw = lambda nbytes, t: nbytes / (t * 1e-3) / 1e9 * (world - 1) / world  # noqa: E731
    ops = 2 * 2.0 * T * hd * F
    # bit-exactness of the sharded FFN against the single-GPU FFN on rank 0's rows is covered by
    # tests/test_gpu_dist.py and tests/test_dist_cpu.py (gloo); here: timing only
    return {"workload": "BERT-large FFN block (h 1024, F 4096) over 256 x 512 tokens, column-parallel x"
                        f"{world} (configs[3])",
            "ms_total": round(tot, 4), "ffn_tops": round(ops / (tot * 1e-3) / 1e12, 1),
            "stages_ms": {k: round(v, 4) for k, v in ms.items()},
            "allgather_int4": {"bytes": int(g1), "busbw_gbs": round(busbw(g1, ms["allgather_int4"]), 1)},
            "allgather_f32": {"bytes": int(g2), "busbw_gbs": round(busbw(g2, ms["allgather_f32"]), 1)},
            "nvlink_ref_gbs": 770.0, "collective": "NCCL all_gather_into_tensor (torch.distributed)",
            "fused_allgather": fused}


def small_configs(torch, dev, pk, regime):
    """BASELINE.json configs[0] (one W4A4 linear M=128, K=N=768, per-tensor
    act scale + per-channel weight scale, bias, fp32 out) and configs[1]
    (BERT-base W4A4 layer, batch 1 x seq 128), each the mean of 100 rounds
    (P:252), graph-timed; everything is L2-resident at these sizes."""
    import synth
    from paper_2203_13483_b200 import mkq as M
    from paper_2203_13483_b200 import model
    out = {}
    Mr, K, N = 128, 768, 768
    x = torch.from_numpy(synth.activations(Mr, K, seed=0)).to(dev)
    w = torch.from_numpy(synth.weight(N, K, seed=1)).to(dev)
    b = torch.from_numpy(synth.bias(N, 1)).to(dev)
    wq, sw = model.prepare_weight(w, 4)
    s_a = 0.5558
    a = M.mkq_quantize_pack(x, torch.tensor([s_a], device=dev), 4, -8, 7)
    y = torch.empty((Mr, N), dtype=torch.float32, device=dev)
    f = lambda st: M.mkq_gemm_w4a4(a, wq, s_a, sw, b, mode=M.OUT_F32, out=y, stream=st)  # noqa: E731
    t1 = graph_time(torch, f, dev, reps=100, inner=1)
    t100 = graph_time(torch, f, dev, reps=100, inner=100)
    ops = 2.0 * Mr * N * K
    nbytes = Mr * K / 2 + N * K / 2 + Mr * N * 4 + 8 * N
    i8 = pk["int8_tops_burst"] if regime == "burst" else pk["int8_tops_sustained"]
    out["c1_linear_m128_k768_n768"] = {
        "us_per_call_single_graph_replay": round(t1 * 1e3, 2), "us_per_call_back_to_back": round(t100 * 1e3, 2),
        "tops": round(ops / (t100 * 1e-3) / 1e12, 2), "frac_int8_peak": round(ops / (t100 * 1e-3) / 1e12 / i8, 4),
        "gbs": round(nbytes / (t100 * 1e-3) / 1e9, 1), "frac_hbm": round(nbytes / (t100 * 1e-3) / 1e9 / pk["hbm_gbs"], 4),
        "bound": "latency (0.74 MB, 0.15 G ops: t_TC 0.03 us, t_HBM 0.1 us vs ~2 us launch+pipeline fill)"}
    h, H, Fh, S = 768, 12, 3072, 128
    p = synth.layer_params(h, H, Fh, 0)
    L = model.build_layer(p, 4, dev)
    model.calibrate(L, torch.from_numpy(synth.hidden_states(8, S, h, seed=1000000)).to(dev), 8, S)
    hin = torch.from_numpy(synth.hidden_states(1, S, h, seed=1)).to(dev)
    ho = torch.empty_like(hin)
    ws = torch.empty(L.workspace_size(S), dtype=torch.uint8, device=dev)
    g = lambda st: M.mkq_bert_layer(L, hin, 1, S, None, h_out=ho, ws=ws, stream=st)  # noqa: E731
    tl1 = graph_time(torch, g, dev, reps=100, inner=1)
    tl = graph_time(torch, g, dev, reps=100, inner=20)
    out["c2_bert_base_layer_b1_s128"] = {
        "us_per_layer_single_graph_replay": round(tl1 * 1e3, 2), "us_per_layer_back_to_back": round(tl * 1e3, 2),
        "effective_tops": round(linear_ops(S, h, Fh) / (tl * 1e-3) / 1e12, 2), "kernels_per_layer": 6 if L.fused_ln(S) else 8,
        "bound": f"latency: {6 if L.fused_ln(S) else 8} dependent kernels at M = 128 (PDL overlaps prologues)"}
    return out


def c3_encoder(torch, dev, reps=20):
    """BASELINE.json configs[2]: BERT-base 12-layer encoder, batch 32 x seq
    128 (4096 tokens), mixed precision per P:243 (layers 1-6 W8A8, 7-12
    W4A4; model.bit_plan(12, 6)), plus the all-W4A4 and all-W8A8 stacks;
    one CUDA graph per stack, mean of `reps` replays (single GPU; the
    row-sharded multi-GPU form runs 32/g sequences per rank)."""
    import synth
    from paper_2203_13483_b200 import model
    h, H, F, B, S = 768, 12, 3072, 32, 128
    T = B * S
    hin = torch.from_numpy(synth.hidden_states(B, S, h, seed=1)).to(dev)
    res = {"tokens": T, "batch": B, "seq": S}
    for name, plan in (("mixed_6w8_6w4", model.bit_plan(12, 6)), ("all_w4a4", [4] * 12), ("all_w8a8", [8] * 12)):
        layers = []
        for i, bits in enumerate(plan):
            p = synth.layer_params(h, H, F, i)
            L = model.build_layer(p, bits, dev)
            model.calibrate(L, torch.from_numpy(synth.hidden_states(4, S, h, seed=1000000 + i)).to(dev), 4, S)
            layers.append(L)
        out = torch.empty_like(hin)
        # fused glue (LN2 writes the next layer's codes, NEXT(4)) and, for the
        # paper's mixed plan, the unfused stack for comparison
        for fuse in ((True, False) if name.startswith("mixed") else (True,)):
            enc = model.Encoder(layers, fuse_codes=fuse)
            ms = graph_time(torch, lambda st: enc(hin, B, S, out=out, stream=st), dev, reps=reps)
            if fuse:
                res[name] = {"plan": "".join(str(b) for b in plan), "ms": round(ms, 4),
                             "tops": round(12 * linear_ops(T, h, F) / (ms * 1e-3) / 1e12, 1),
                             "compression_vs_fp32": round(model.compression_ratio(plan), 3),
                             "fused_layer_codes": True}
            else:
                res[name]["unfused_ms"] = round(ms, 4)
    return res


def qat_calibration(torch, M, x, stream, pk, reps=10):
    """SURVEY §8f NEXT(3)/(4) kernels on the bench's layer input (T x hidden
    fp32, > L2): mkq_fake_quant with every output (y, STE grad_x, STE/MSE
    grad_s; 16 algorithmic B/element) and mkq_act_scale (the P:72 percentile
    calibration; 3 radix passes = 12 B/element), CUDA-event timed."""
    gy = torch.randn_like(x)
    sc = torch.tensor([0.5558], device=x.device)
    ws = torch.empty(int(M.lib().mkq_fake_quant_workspace_size(x.numel())), dtype=torch.uint8, device=x.device)
    res = {}
    with torch.cuda.stream(stream):
        for name, fn, bpe in (
                ("fake_quant_grad", lambda: M.mkq_fake_quant(x, sc, -8, 7, grad_y=gy, ws=ws, stream=stream), 16),
                ("act_scale_p99.99", lambda: M.mkq_act_scale(x, 7.0, 0.9999, stream=stream), 12)):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            gbs = bpe * x.numel() / (us * 1e-6) / 1e9
            res[name] = {"us": round(us, 1), "elements": x.numel(), "algorithmic_bytes_per_element": bpe,
                         "gbs": round(gbs, 1), "bound": "hbm", "frac": round(gbs / pk["hbm_gbs"], 4)}
    del gy
    return res


def compare_float_layers(torch, p, dev, int4_ms, args):
    """fp32 (TF32 off) and bf16 torch/cuBLAS BERT-large layer on the same
    shape, for the paper's int4-vs-fp32 speedup methodology (Table 2)."""
    import torch.nn.functional as Fn
    B, S, hd, H, F = CFG["batch"], CFG["seq"], CFG["hidden"], CFG["heads"], CFG["ffn"]
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    out = {}
    for dt in (torch.float32, torch.bfloat16):
        W = {k: torch.from_numpy(getattr(p, k)).to(dev, dt) for k in
             ("w_qkv", "b_qkv", "w_o", "b_o", "w_1", "b_1", "w_2", "b_2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")}
        chunk = 32
        x = torch.randn(chunk * S, hd, device=dev, dtype=dt)

        def layer(h):
            qkv = Fn.linear(h, W["w_qkv"], W["b_qkv"]).view(chunk, S, 3, H, 64)
            q, k, v = qkv.unbind(2)
            a = Fn.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2))
            a = a.transpose(1, 2).reshape(chunk * S, hd)
            h1 = Fn.layer_norm(Fn.linear(a, W["w_o"], W["b_o"]) + h, (hd,), W["ln1_g"], W["ln1_b"], 1e-12)
            f = Fn.linear(Fn.gelu(Fn.linear(h1, W["w_1"], W["b_1"])), W["w_2"], W["b_2"])
            return Fn.layer_norm(f + h1, (hd,), W["ln2_g"], W["ln2_b"], 1e-12)

        for _ in range(2):
            layer(x)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 2
        e0.record()
        for _ in range(reps):
            for _c in range(B // chunk):
                layer(x)
        e1.record()
        torch.cuda.synchronize(dev)
        out["fp32_layer_ms" if dt == torch.float32 else "bf16_layer_ms"] = round(e0.elapsed_time(e1) / reps, 3)
        del W, x
    out["int4_layer_ms"] = round(int4_ms, 3)
    out["speedup_int4_vs_fp32"] = round(out["fp32_layer_ms"] / int4_ms, 2)
    out["speedup_int4_vs_bf16"] = round(out["bf16_layer_ms"] / int4_ms, 2)
    out["paper_context"] = "MKQ-BERT Table 2 (P:250-264): int4 15x vs fp32 for one BERT-base layer, NVIDIA T4, BS64"
    torch.backends.cuda.matmul.allow_tf32 = True
    return out


# ------------------------------------------------------------------ paper Table 2 workload
TABLE2 = [(16, 440), (16, 537), (16, 681), (64, 1691), (64, 2011), (64, 2298)]   # P:258-264 (BS, valid tokens)
TABLE2_T4_US = {(16, 440): (1380, 213.1, 160.5), (16, 537): (1845, 245.7, 179.3), (16, 681): (2690, 260.9, 196.5),
                (64, 1691): (6398, 567.4, 428.8), (64, 2011): (7185, 628.4, 490.1), (64, 2298): (7897, 669.9, 533.4)}


def table2(torch, dev, reps=50):
    """Paper Table 2 methodology on B200: one BERT-base layer
    (h 768, 12 heads, FFN 3072) over BS sequences of max length 128 with the
    given number of valid (non-padding) tokens, packed (cu_seqlens, R13);
    int4 (W4A4) and int8 (W8A8) layers through mkq_bert_layer captured in a
    CUDA graph, fp32 (TF32 off) torch/cuBLAS layer on the valid tokens;
    mean of `reps` CUDA-graph replays / eager runs."""
    import synth
    import torch.nn.functional as Fn
    from paper_2203_13483_b200 import mkq as M
    from paper_2203_13483_b200 import model
    h, H, F, S = 768, 12, 3072, 128
    p = synth.layer_params(h, H, F, 0)
    layers = {}
    for key, bits, ia in (("int4", 4, False), ("int8", 8, False), ("int4_int_attention", 4, True)):
        L = model.build_layer(p, bits, dev)
        hc = torch.from_numpy(synth.hidden_states(8, S, h, seed=1000000)).to(dev)
        model.calibrate(L, hc, 8, S, int_attention=ia)
        layers[key] = L
    W = {k: torch.from_numpy(getattr(p, k)).to(dev) for k in
         ("w_qkv", "b_qkv", "w_o", "b_o", "w_1", "b_1", "w_2", "b_2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")}
    torch.backends.cuda.matmul.allow_tf32 = False
    rows = []
    for bs, valid in TABLE2:
        lens = synth.varlen_seqlens(bs, valid, S, seed=bs + valid)
        cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), device=dev)
        hin = torch.from_numpy(synth.hidden_states(1, valid, h, seed=1)).to(dev)
        res = {"bs": bs, "valid_tokens": valid}
        for key in ("int4", "int8", "int4_int_attention"):
            L = layers[key]
            out = torch.empty_like(hin)
            ws = torch.empty(L.workspace_size(valid), dtype=torch.uint8, device=dev)
            st = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(st):
                for _ in range(3):
                    M.mkq_bert_layer(L, hin, bs, S, cu, h_out=out, ws=ws, stream=st)
            torch.cuda.synchronize(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                M.mkq_bert_layer(L, hin, bs, S, cu, h_out=out, ws=ws, stream=st)
            g.replay()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize(dev)
            res[f"{key}_us"] = round(e0.elapsed_time(e1) / reps * 1e3, 1)
        # fp32 torch/cuBLAS layer on the VALID tokens (like for like with the packed int4 layer):
        # linears, GELU and LayerNorms on the packed [valid, h] rows; attention (a small share at
        # s <= 128) on the padded [bs, 128] batch with a key mask, pad / unpad gathers included
        mask = torch.zeros(bs, S, dtype=torch.bool, device=dev)
        for i, Lq in enumerate(lens):
            mask[i, :Lq] = True
        idx = mask.view(-1).nonzero().squeeze(1)
        am = torch.where(mask[:, None, None, :], 0.0, float("-inf"))
        x = torch.from_numpy(synth.hidden_states(1, valid, h, seed=1)).to(dev)

        def layer32(xx):
            qkv = Fn.linear(xx, W["w_qkv"], W["b_qkv"])
            pad = torch.zeros(bs * S, 3 * h, device=dev).index_copy_(0, idx, qkv).view(bs, S, 3, H, 64)
            q, k, v = pad.unbind(2)
            a = Fn.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), attn_mask=am)
            a = a.transpose(1, 2).reshape(bs * S, h).index_select(0, idx)
            h1 = Fn.layer_norm(Fn.linear(a, W["w_o"], W["b_o"]) + xx, (h,), W["ln1_g"], W["ln1_b"], 1e-12)
            f = Fn.linear(Fn.gelu(Fn.linear(h1, W["w_1"], W["b_1"])), W["w_2"], W["b_2"])
            return Fn.layer_norm(f + h1, (h,), W["ln2_g"], W["ln2_b"], 1e-12)

        for _ in range(3):
            layer32(x)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            layer32(x)
        e1.record()
        torch.cuda.synchronize(dev)
        res["fp32_us"] = round(e0.elapsed_time(e1) / reps * 1e3, 1)
        res["int4_vs_fp32"] = round(res["fp32_us"] / res["int4_us"], 2)
        res["int4_vs_int8"] = round(res["int8_us"] / res["int4_us"], 2)
        t4 = TABLE2_T4_US[(bs, valid)]
        res["paper_T4_us_fp32_int8_int4"] = list(t4)
        rows.append(res)
    torch.backends.cuda.matmul.allow_tf32 = True
    return rows


# ------------------------------------------------------------------ oracle (CPU) arm
def host_info():
    """nproc, the affinity mask size and the CPU model of the host the oracle ran on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"nproc": os.cpu_count(), "affinity_cpus": aff, "cpu_model": model, "threads_used": 1}


def cpu_baseline(sample_seqs=1):
    """The oracle as it stands, on the host cores, over a bounded sample of
    the same workload (whole sequences of the BERT-large layer)."""
    import oracle
    from oracle import layer as OL
    import synth
    hd, H, F, S = CFG["hidden"], CFG["heads"], CFG["ffn"], CFG["seq"]
    p = synth.layer_params(hd, H, F, 0)
    W = OL.LayerWeights(hd, H, F, 4, OL.prepare_weight(p.w_qkv, p.b_qkv, 4), OL.prepare_weight(p.w_o, p.b_o, 4),
                        OL.prepare_weight(p.w_1, p.b_1, 4), OL.prepare_weight(p.w_2, p.b_2, 4),
                        p.ln1_g, p.ln1_b, p.ln2_g, p.ln2_b)
    W.s_qkv_in = W.s_o_in = W.s_ffn1_in = np.float32(3.8906 / 7)
    W.s_ffn2_in = np.float32(0.5)
    h = synth.hidden_states(sample_seqs, S, hd, seed=0)
    oracle.build()
    t0 = time.perf_counter()
    OL.bert_layer(h, W, [S] * sample_seqs)
    dt = time.perf_counter() - t0
    T = sample_seqs * S
    return {"value": round(linear_ops(T, hd, F) / dt / 1e12, 6), "unit": "TOPS", "cores": 1, "kind": "oracle",
            "host": host_info(),
            "sample": f"{sample_seqs} x {S}-token sequence(s) of the BERT-large W4A4 layer (oracle/: scalar C int "
                      f"GEMM + fp64 NumPy glue, single thread), {dt:.2f} s",
            "seconds": round(dt, 3)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    vals = []
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_baseline(1)
    for _ in range(args.steps):
        vals.append(cpu_baseline(1))
    v = float(np.mean([c["value"] for c in vals]))
    sec = float(np.mean([c["seconds"] for c in vals]))
    res = {
        "impl": "reference",
        "metric": "W4A4 GEMM TOPS (effective: layer linear-GEMM int ops / BERT int4 layer time)",
        "value": round(v, 6), "unit": "TOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 1), "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "s4 x s4 -> s32 (scalar C), fp64 glue", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": "1 sequence of 512 tokens per step"},
        "cpu_baseline": {"value": round(v, 6), "unit": "TOPS", "cores": 1, "kind": "oracle",
                         "sample": "1 x 512-token sequence per step", "host": host_info()},
        "e2e": {"value": round(v, 6), "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-compare", action="store_true", help="skip the fp32/bf16 torch comparison layer")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    ap.add_argument("--no-table2", action="store_true", help="skip the paper Table 2 (BERT-base varlen) rows")
    ap.add_argument("--no-extras", action="store_true", help="only the headline line (no single-GPU extra sections)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the configs[3] batch (256 x 512) sharded over the ranks (default); "
                         "weak: a full batch per rank")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
