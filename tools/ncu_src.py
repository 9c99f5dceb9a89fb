"""Summarise an ncu --set full --import-source capture (diagnostics):
duration, issue, and the CUDA source lines with the most warp-stall samples,
with their dominant stall reasons.   python tools/ncu_src.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    for r in csv.reader(io.StringIO(det)):
        if len(r) > 3 and r[-3] in ("Duration", "Issue Slots Busy", "Executed Instructions", "SM Frequency",
                                     "Registers Per Thread", "Block Size"):
            print(f"{r[-3]}: {r[-1]} {r[-2]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, out, tot = None, [], 0
    hdr = None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r) if i >= 2}
            continue
        if hdr and r and r[0] != "" and len(r) > 7:
            s = int(r[6]) if r[6].isdigit() else 0
            tot += s
            if s:
                st = {h[6:]: int(r[i]) for h, i in hdr.items()
                      if h.startswith("stall_") and "Not Issued" not in h and r[i].isdigit() and int(r[i]) >= 0.15 * s}
                out.append((s, cur, r[0], r[1].strip()[:70], st, r[7]))
    print("total samples", tot)
    for o in sorted(out, reverse=True)[:top]:
        print(f"{o[0]:6d} {100*o[0]/tot:5.1f}% {o[1]}:{o[2]} exec={o[5]} {o[3]!r} {o[4]}")


if __name__ == "__main__":
    main()
