"""Per-source-line warp-stall summary of an ncu report (diagnostics).
usage: python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
hdr = None
out = []
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            out.append((int(r[4]), fname, r[0], r[1].strip()[:60], r))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
print(f"total samples {tot}")
for s, f, ln, src, r in sorted(out, key=lambda o: -o[0])[:top]:
    reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:3]
    rs = " ".join(f"{n}:{v}" for v, n in reasons if v)
    print(f"{100*s/tot:5.1f}% {f[:20]:20s}:{ln:>4s} {src:60s} {rs}")
