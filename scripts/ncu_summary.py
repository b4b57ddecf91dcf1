#!/usr/bin/env python
"""Summarise an ncu report: key throughput metrics + top stalled SASS lines per kernel."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            for k in KEYS:
                if h.endswith(k):
                    d[k] = (v, u)
        yield d


def top_sass(rep, n):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = {"rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    for b in blocks:
        h = b["hdr"]
        i_s, i_src, i_ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
        tot = sum(float(r[i_s] or 0) for r in b["rows"]) or 1
        rows = sorted(b["rows"], key=lambda r: -float(r[i_s] or 0))[:n]
        yield [(f"{100*float(r[i_s] or 0)/tot:5.1f}%", r[i_ex], r[i_src][:80]) for r in rows]


if __name__ == "__main__":
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    for i, d in enumerate(raw(rep)):
        print(f"--- launch {i}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][0]} {d[k][1]}")
    for i, rows in enumerate(top_sass(rep, n)):
        print(f"--- top stalls, kernel {i}")
        for r in rows:
            print("  ", *r)
