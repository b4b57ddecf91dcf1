#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples of an ncu report (needs -lineinfo + --import-source on).
  python scripts/ncu_lines.py report.ncu-rep [n]"""
import csv, io, subprocess, sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, rows, fname = None, [], ""
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] and len(r) == len(hdr):
        rows.append((fname, r))
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for _, r in rows if r[i_s] not in ("", "-")) or 1
def f(x):
    try: return float(x)
    except ValueError: return 0.0
for fn, r in sorted(rows, key=lambda x: -f(x[1][i_s]))[:n]:
    print(f"{100 * f(r[i_s]) / tot:5.1f}% {r[i_e]:>10} {fn}:{r[0]} {r[1].strip()[:100]}")
