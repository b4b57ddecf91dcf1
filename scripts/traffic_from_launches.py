#!/usr/bin/env python
"""profiles/traffic.json from the ncu launch list of `bench.py --launch-list`
(gpu__time_duration + dram__bytes_{read,write} per tm_gemm_kernel launch, one
sweep): DRAM bytes per launch of each kernel group of the sweep, which bench.py
reports as roofline.traffic next to the algorithmic bytes.
  python scripts/traffic_from_launches.py gpurun_out/<tag>/launches.csv profiles/traffic.json
"""
import collections
import csv
import json
import sys


def main(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    launches = [d for d in per.values() if any(k in d["name"] for k in ("tm_gemm_kernel", "tm_rowband_kernel", "tm_halo_kernel"))]
    # sweep order (bench.build_sweep): 53 conv launches, FFN (2), QK^T, PV
    groups = [("conv", 53), ("ffn", 2), ("attn", 2)]
    if len(launches) != sum(n for _, n in groups):
        raise SystemExit(f"expected 57 tm_gemm / rowband / halo launches (one sweep), got {len(launches)}")
    out, i = {}, 0
    for g, n in groups:
        ls = launches[i:i + n]
        i += n
        by = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ls)
        t = sum(d.get("gpu__time_duration.sum", 0) for d in ls)
        out[g] = {"launches": n, "dram_bytes_per_launch": by / n, "ncu_us_per_launch": t / n / 1e3}
    out["source"] = f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum ({src})"
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
