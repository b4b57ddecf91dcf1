#!/usr/bin/env python
"""BASELINE configs[0] lines alone (fp32 CUDA-core, tf32, bf16 forms of 1024^3 + bias + ReLU)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch
    import bench
    print(json.dumps(bench.config1_lines(torch, torch.device("cuda", 0), bench.peaks()[0], None)))
