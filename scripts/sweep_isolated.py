#!/usr/bin/env python
"""Per-workload device time of the bench sweep measured in isolation (a CUDA
graph of 20 back-to-back launches of the same bound exec), summed and compared
with the whole-sweep graph: the difference is the cost of transitions between
different kernels (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2210_09603_b200 import Graph
    from paper_2210_09603_b200.tuning import TuningCache
    dev = torch.device("cuda", 0)
    items, _ = bench.build_sweep(torch, dev, seed=1234, tuner=TuningCache(os.path.join(ROOT, "tuning_cache.json")),
                                 tune_mode="auto", log=None)
    total = 0.0
    for it in items:
        g = Graph([it["exec"]] * 20)
        g.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        total += ms
        print(f"{it['name']:12s} {ms * 1e3:7.1f} us  {it['flops'] / ms / 1e9:7.1f} TFLOP/s")
    sweep = Graph([it["exec"] for it in items])
    for _ in range(3):
        sweep.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sweep.launch()
    e1.record()
    torch.cuda.synchronize()
    print(f"sum of isolated {total * 1e3:.1f} us; sweep graph {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
