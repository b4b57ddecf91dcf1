#!/usr/bin/env python
"""Per-stage table of the ResNet-50 chain's graph replay from an ncu launch list
(scripts/chain_once.py under ncu --metrics gpu__time_duration.sum,dram__bytes_*).
The replay is the last 56 product launches of the process (the eager warm-up pass
precedes it).  ncu serialises launches and runs them cold, so absolute times exceed
the graph's; the shares are what to read.
  python scripts/chain_launch_table.py chain_launches.csv > profiles/r02/chain_launches.md"""
import csv
import io
import sys

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2210_09603_b200 import workloads as W  # noqa: E402

rows = {}
text = open(sys.argv[1]).read()
body = text[text.index('"ID"'):]
for r in csv.DictReader(io.StringIO(body)):
    k = rows.setdefault(int(r["ID"]), {"name": r["Kernel Name"], "grid": r["Grid Size"]})
    k[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ours = [rows[i] for i in sorted(rows) if "tmb::" in rows[i]["name"] or "tmb_rule" in rows[i]["name"]]
stages = W.resnet50_stages()
rep = ours[-len(stages):]
tot = sum(k["gpu__time_duration.sum"] for k in rep)
print("| stage | kind | kernel | grid | time µs | share | DRAM MB |")
print("|---|---|---|---|---|---|---|")
fam = {}
for st, k in zip(stages, rep):
    name = k["name"].split("(")[0].replace("void ", "").replace("tmb::", "")
    t = k["gpu__time_duration.sum"] / 1e3
    mb = (k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)) / 1e6
    f = fam.setdefault(st.kind if st.kind != "conv" else ("conv c3 (residual)" if st.res else "conv"), [0, 0.0, 0.0])
    f[0] += 1
    f[1] += t
    f[2] += mb
    print(f"| {st.dst} | {st.kind} | `{name}` | {k['grid']} | {t:.1f} | {100 * t * 1e3 / tot:.1f}% | {mb:.1f} |")
print()
print(f"total {tot / 1e3:.1f} µs over {len(rep)} launches (ncu, serialised, cold)")
print()
print("| family | launches | µs | share | DRAM MB |")
print("|---|---|---|---|---|")
for f, (n, t, mb) in sorted(fam.items(), key=lambda x: -x[1][1]):
    print(f"| {f} | {n} | {t:.1f} | {100 * t * 1e3 / tot:.1f}% | {mb:.1f} |")
