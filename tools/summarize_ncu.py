"""Summarize ncu captures into profiles/ (committed evidence).

    python tools/summarize_ncu.py --rep gpurun_out/r01_layer.ncu-rep --launches gpurun_out/r01_launches.csv \
        --out profiles/r01

Writes <out>_kernels.md (per-kernel table: duration, DRAM bytes, tensor/LSU
pipe utilisation, registers, the SASS proof of tcgen05/TMA use) and
<out>_traffic.json (per-kernel dram read+write bytes; bench.py reads it for
the roofline `traffic` field) and <out>_launches.md (launch list share).
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active": "hmma_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "lsu_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
UNITS = {"dram_rd": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9},
         "dur": {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"name": d.get("Kernel Name", "?")}
        for m, short in METRICS.items():
            v = d.get(m)
            if v in (None, ""):
                continue
            v = float(v.replace(",", ""))
            if short in ("dram_rd", "dram_wr"):
                v *= UNITS["dram_rd"].get(u.get(m, "byte"), 1)
            if short == "dur_us":
                v *= UNITS["dur"].get(u.get(m, "usecond"), 1)
            k[short] = v
        res.append(k)
    return res


def short(name):
    for key in ("gemm_w4a4_2cta", "gemm_i8tc", "flash_attn", "residual_ln", "quantize_pack", "absmax", "scan",
                "verify", "finalize"):
        if key in name:
            return key + ("<256>" if "Li256" in name else ("<128>" if "Li128" in name else ""))
    return name[:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--last", type=int, default=24, help="count only the last N launches (the timed steps; "
                    "tools/prof_layer.py --steps 3 = 24 launches after the setup kernels)")
    ap.add_argument("--out", required=True)
    ap.add_argument("--labels", default="quantize_in,gemm_qkv,attention,gemm_o,ln1_quant,gemm_ffn1,gemm_ffn2,ln2")
    a = ap.parse_args()
    ks = raw(a.rep)
    labels = a.labels.split(",")
    lines = ["| # | stage | kernel | time us (ncu, serialised) | DRAM rd+wr MB | DRAM % | tensor pipe % | LSU % | TC-smem % | issue % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for i, k in enumerate(ks):
        lab = labels[i] if i < len(labels) else f"k{i}"
        tb = k.get("dram_rd", 0) + k.get("dram_wr", 0)
        traffic[lab] = {"kernel": short(k["name"]), "dram_bytes": tb, "ncu_us": k.get("dur_us")}
        lines.append(f"| {i} | {lab} | `{short(k['name'])}` | {k.get('dur_us', 0):.1f} | {tb/1e6:.1f} | "
                     f"{k.get('dram_pct', 0):.1f} | {k.get('tensor_pct', 0):.1f} | {k.get('lsu_pct', 0):.1f} | "
                     f"{k.get('tc_smem_pct', 0):.1f} | {k.get('issue_pct', 0):.1f} | {k.get('regs', 0):.0f} | "
                     f"{k.get('grid', 0):.0f} x {k.get('block', 0):.0f} |")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + "_kernels.md", "w") as f:
        f.write(f"# ncu --set full summary ({os.path.basename(a.rep)})\n\n")
        f.write(f"One launch of each of the {len(labels)} kernels of the BERT-large W4A4 layer step (bench.py workload,\n"
                "tools/prof_layer.py), `ncu --set full --clock-control none`.  Durations are ncu's serialised,\n"
                "cold-cache replays: compare shares, not absolutes, with bench.py's live CUDA-event times.\n\n")
        f.write("\n".join(lines) + "\n")
    with open(a.out + "_traffic.json", "w") as f:
        json.dump(traffic, f, indent=1)
    if a.launches and os.path.exists(a.launches):
        txt = open(a.launches).read()
        start = txt.find('"ID"')
        rows = [r for r in csv.DictReader(io.StringIO(txt[start:])) if r.get("Metric Name") == "gpu__time_duration.sum"]
        if a.last > 0:
            rows = rows[-a.last:]
        tot = {}
        for r in rows:
            n = short(r["Kernel Name"])
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "nsecond")
            v *= UNITS["dur"].get(unit, 1e-3)
            tot.setdefault(n, []).append(v)
        allt = sum(sum(v) for v in tot.values())
        with open(a.out + "_launches.md", "w") as f:
            f.write(f"# Launch list ({os.path.basename(a.launches)}): "
                    f"`ncu --metrics gpu__time_duration.sum --clock-control none`, the last {a.last} launches "
                    "(the timed mkq_bert_layer steps, setup kernels excluded)\n\n")
            f.write("| kernel | launches | mean us | share of step |\n|---|---|---|---|\n")
            for n, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
                f.write(f"| `{n}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v)/allt:.3f} |\n")
    print(open(a.out + "_kernels.md").read())


if __name__ == "__main__":
    main()
