"""Per-stage device time of a BERT-base layer at Table-2 sizes, each stage
captured 20x back to back in one CUDA graph (steady-state per-launch time,
no host gaps).  Env: BITS, T, BS, MKQ_SMALL_M."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2203_13483_b200 import mkq as M, model
bits = int(os.environ.get("BITS", 4)); T = int(os.environ.get("T", 440)); bs = int(os.environ.get("BS", 16))
h, H, F, S = 768, 12, 3072, 128
p = synth.layer_params(h, H, F, 0)
L = model.build_layer(p, bits, "cuda")
model.calibrate(L, torch.from_numpy(synth.hidden_states(8, S, h, seed=1000000)).cuda(), 8, S)
lens = synth.varlen_seqlens(bs, T, S, seed=bs + T)
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), device="cuda")
x = torch.from_numpy(synth.hidden_states(1, T, h, seed=1)).cuda()
lo, hi = model.act_range(bits); t = L.t; s = L.scales
gemm = M.mkq_gemm_w4a4 if bits == 4 else M.mkq_gemm_w8a8
cb = h // 2 if bits == 4 else h
dt = torch.uint8 if bits == 4 else torch.int8
codes = torch.empty((T, cb), dtype=dt, device="cuda")
qkv = torch.empty((T, 3 * h), dtype=torch.float16, device="cuda")
oa = torch.empty((T, cb), dtype=dt, device="cuda")
o = torch.empty((T, h), device="cuda"); h1 = torch.empty_like(o); c1 = torch.empty_like(codes)
a2 = torch.empty((T, F // 2 if bits == 4 else F), dtype=dt, device="cuda"); f = torch.empty_like(o); out = torch.empty_like(o)
sq = torch.tensor([s["s_qkv_in"]], device="cuda")
st = torch.cuda.Stream()
calls = [("quant", lambda: M.mkq_quantize_pack(x, sq, bits, lo, hi, out=codes, stream=st)),
         ("qkv", lambda: gemm(codes, t["w_qkv"], s["s_qkv_in"], t["sw_qkv"], t["b_qkv"], mode=M.OUT_F16, out=qkv, K=h, stream=st)),
         ("attn", lambda: M.mkq_attention(qkv, H, bs, S, cu, mode=M.OUT_I4 if bits == 4 else M.OUT_I8, s_out=s["s_o_in"], qmin=lo, qmax=hi, out=oa, stream=st)),
         ("o", lambda: gemm(oa, t["w_o"], s["s_o_in"], t["sw_o"], t["b_o"], mode=M.OUT_F32, out=o, K=h, stream=st)),
         ("ln1", lambda: M.mkq_residual_layernorm(o, x, t["ln1_g"], t["ln1_b"], 1e-12, bits=bits, s_q=s["s_ffn1_in"], qmin=lo, qmax=hi, y=h1, q=c1, stream=st)),
         ("ffn1", lambda: gemm(c1, t["w_1"], s["s_ffn1_in"], t["sw_1"], t["b_1"], mode=M.OUT_I4 if bits == 4 else M.OUT_I8, gelu=True, s_out=s["s_ffn2_in"], qmin=lo, qmax=hi, out=a2, K=h, requant_table=L.table, stream=st)),
         ("ffn2", lambda: gemm(a2, t["w_2"], s["s_ffn2_in"], t["sw_2"], t["b_2"], mode=M.OUT_F32, out=f, K=F, stream=st)),
         ("ln2", lambda: M.mkq_residual_layernorm(f, h1, t["ln2_g"], t["ln2_b"], 1e-12, y=out, stream=st))]
if bits == 4:   # the fused W^A + LN1 / W^2 + LN2 kernels (mkq_gemm_residual_ln; not in stage_sum)
    lnws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    calls += [("o_ln1*", lambda: M.mkq_gemm_residual_ln(oa, t["w_o"], s["s_o_in"], t["sw_o"], t["b_o"], x, t["ln1_g"], t["ln1_b"], 1e-12, K=h, q_bits=4, s_q=s["s_ffn1_in"], qmin=lo, qmax=hi, y=h1, q=c1, stream=st)),
              ("ffn2_ln2*", lambda: M.mkq_gemm_residual_ln(a2, t["w_2"], s["s_ffn2_in"], t["sw_2"], t["b_2"], h1, t["ln2_g"], t["ln2_b"], 1e-12, K=F, y=out, stream=st))]
R = 20
res = {}
with torch.cuda.stream(st):
    for name, c in calls:
        for _ in range(3):
            c()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(R):
                c()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) * 1e3 / (10 * R), 2)
# whole layer graph
ws = torch.zeros(L.workspace_size(T), dtype=torch.uint8, device="cuda")
with torch.cuda.stream(st):
    for _ in range(3):
        M.mkq_bert_layer(L, x, bs, S, cu, h_out=out, ws=ws, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(R):
            M.mkq_bert_layer(L, x, bs, S, cu, h_out=out, ws=ws, stream=st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
res["layer_x20"] = round(e0.elapsed_time(e1) * 1e3 / (10 * R), 2)
print(f"bits={bits} T={T} small={os.environ.get('MKQ_SMALL_M', 'auto')}:", res, "stage_sum", round(sum(v for k, v in res.items() if k != 'layer_x20' and not k.endswith('*')), 1), flush=True)
# kernel-switch cost (diagnostics): pairs of different stages alternating in one graph vs each alone
if os.environ.get("PAIRS"):
    names = [n for n, _ in calls]
    fn = dict(calls)
    for a_, b_ in [("qkv", "o"), ("o", "ffn2"), ("qkv", "ffn2"), ("ln1", "ln2"), ("quant", "ln2")]:
        with torch.cuda.stream(st):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(R // 2):
                    fn[a_](); fn[b_]()
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                g.replay()
            e1.record(st)
            torch.cuda.synchronize()
        pair_us = e0.elapsed_time(e1) * 1e3 / (10 * (R // 2))
        print(f"pair {a_}+{b_}: {pair_us:.2f} us alternating vs {res[a_] + res[b_]:.2f} alone-sum", flush=True)
