#!/usr/bin/env python
"""One-line-per-capture summary of ncu --set full reports (for profiles/):
duration, SM clock, tensor-pipe utilisation, DRAM / L2 bytes and throughput,
achieved TFLOP/s from the GEMM flops (sm__ops_path_tensor...utchmma... counts MACs*2).
  python scripts/ncu_report.py gpurun_out/<tag>/*.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "dur",
    "gpc__cycles_elapsed.max.per_second": "clk",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum": "tc_ops",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "lts__t_bytes.sum": "l2_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def report(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for h, u, v in zip(hdr, units, r):
            for k, name in WANT.items():
                if h == k:
                    try:
                        d[name] = float(v.replace(",", "")) * SCALE.get(u, 1)
                    except ValueError:
                        d[name] = None
        yield d


def main(paths):
    print("| capture | kernel | grid | regs | duration us | SM GHz | tensor pipe % | TFLOP/s (tc ops) | DRAM MB (rd+wr) | DRAM % | L2 % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        for d in report(p):
            dur = d.get("dur") or float("nan")
            tf = (d.get("tc_ops") or 0) / dur / 1e12 if dur == dur else float("nan")
            dram = ((d.get("dram_rd") or 0) + (d.get("dram_wr") or 0)) / 1e6
            print(f"| {p.split('/')[-1]} | {d['kernel']} | {d.get('grid', 0):.0f} | {d.get('regs', 0):.0f} | "
                  f"{dur * 1e6:.1f} | {(d.get('clk') or 0) / 1e9:.2f} | {d.get('tensor_pct') or 0:.1f} | {tf:.0f} | "
                  f"{dram:.1f} | {d.get('dram_pct') or 0:.1f} | {d.get('l2_pct') or 0:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
