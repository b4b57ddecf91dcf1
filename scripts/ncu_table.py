#!/usr/bin/env python
"""Markdown table of ncu --set full captures (profiles/): duration, SM clock,
tensor-pipe utilisation, achieved tensor TFLOP/s (tcgen05 ops), DRAM bytes and
GB/s with the fraction of the measured HBM peak (MEASURED_PEAKS.json), L2 and
SM throughput.  python scripts/ncu_table.py <reports...>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_report import report  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(paths):
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        hbm = 6555.2
    print(f"| capture | kernel | grid | regs | duration us | SM GHz | tensor pipe % | tensor TFLOP/s | "
          f"DRAM MB | DRAM GB/s | % of {hbm:.0f} GB/s | L2 % | SM % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        for d in report(p):
            dur = d.get("dur") or float("nan")
            tf = (d.get("tc_ops") or 0) / dur / 1e12
            dram = (d.get("dram_rd") or 0) + (d.get("dram_wr") or 0)
            gbs = dram / dur / 1e9
            print(f"| {os.path.basename(p)} | {d['kernel'][:48]} | {d.get('grid') or 0:.0f} | {d.get('regs') or 0:.0f} | "
                  f"{dur * 1e6:.1f} | {(d.get('clk') or 0) / 1e9:.2f} | {d.get('tensor_pct') or 0:.1f} | {tf:.0f} | "
                  f"{dram / 1e6:.1f} | {gbs:.0f} | {100 * gbs / hbm:.1f} | {d.get('l2_pct') or 0:.1f} | "
                  f"{d.get('sm_pct') or 0:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
