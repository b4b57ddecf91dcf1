#!/usr/bin/env python
"""Timeline of the row-band conv kernel (TMB_TRACE=1): python scripts/rb_trace.py [layer]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["TMB_TRACE"] = "1"


def main():
    import numpy as np
    import torch
    from paper_2210_09603_b200 import Plan, ScheduleConfig, workloads as W
    name = sys.argv[1] if len(sys.argv) > 1 else "conv1"
    L = next(x for x in W.RESNET50 if x.name == name)
    B, dev = W.RESNET_BATCH, torch.device("cuda", 0)
    xb = torch.zeros((B, L.h, L.h, 4), device=dev, dtype=torch.bfloat16)
    xb[..., :L.c] = torch.empty((B, L.h, L.h, L.c), device=dev).uniform_(-1, 1).to(torch.bfloat16)
    x = xb.as_strided((B, L.c, L.h, L.h), (L.h * L.h * 4, 1, L.h * 4, 4))
    w = torch.empty((L.f, L.c, L.k, L.k), device=dev).uniform_(-1, 1).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    s, t = torch.rand(L.f, device=dev), torch.rand(L.f, device=dev)
    ho = L.out_hw()
    z = torch.empty((B, L.f, ho, ho), device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    ex = Plan(W.conv_bn_relu_dag(L, B), ScheduleConfig(block_n=64)).bind([x, w, s, t], [z])
    for _ in range(3):
        ex.launch()
    torch.cuda.synchronize()
    tr = ex.trace(0)
    names = ["mma0", "mma1", "epiA", "epiD", "bandR", "bandI", "-"]
    for cta in (0, 1, 77, tr.shape[0] - 1):
        print(f"CTA {cta}")
        for i in range(40):
            row = tr[cta, i, :7]
            if row.any():
                print(f"  tile {i:2d} " + " ".join(f"{n}={v:7d}" for n, v in zip(names, row)))
    last = tr[:, :, 3].max(axis=1)
    print("CTA finish (clk): min", last.min(), "median", int(np.median(last)), "max", last.max())
    mm = tr[:, :, 1] - tr[:, :, 0]
    print("mean MMA issue span per tile", mm[tr[:, :, 1] > 0].mean())


if __name__ == "__main__":
    main()
