"""Attribute spin-wait iterations of an ncu source capture to barriers (diagnostics)."""
import csv, re, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ix = hdr.index("Instructions Executed"); isamp = hdr.index("Warp Stall Sampling (All Samples)")
tot_i = sum(int(r[ix] or 0) for r in data); tot_s = sum(int(r[isamp] or 0) for r in data)
print("total instr", tot_i, "samples", tot_s)
for r in data:
    m = re.search(r"TRYWAIT\S* P\d, \[(R\d+)\+URZ\+(0x[0-9a-f]+)\]", r[1])
    if m and int(r[ix] or 0) > 0:
        print(f"{r[0][-5:]} off={m.group(2)} exec={int(r[ix])} samples={r[isamp]}  {r[1][:80]}")
