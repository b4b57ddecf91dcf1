#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv):
per-kernel launch counts, time share and (when captured) DRAM bytes.
  python scripts/launch_summary.py gpurun_out/<tag>/launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ix["ID"]], r[ix["Kernel Name"]])
        d = per.setdefault(key, {})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), d in per.items():
        short = name.split("(")[0].replace("void ", "")
        a = agg[short]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'time_us':>10s} {'share':>7s} {'dram_MB':>9s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {a[0]:8d} {a[1] / 1e3:10.1f} {a[1] / total:7.1%} {a[2] / 1e6:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
