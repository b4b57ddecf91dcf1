#!/usr/bin/env python
"""BASELINE configs[0] lines alone (fp32 CUDA-core, tf32, bf16 forms of 1024^3 + bias + ReLU);
--large: bench.py's large-shape lines (8192^3 GEMM, batch-256 ResNet 3x3 convs)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch
    import bench
    dev = torch.device("cuda", 0)
    if "--large" in sys.argv:
        print(json.dumps(bench.large_lines(torch, dev, bench.peaks()[0])))
    else:
        print(json.dumps(bench.config1_lines(torch, dev, bench.peaks()[0], None)))
