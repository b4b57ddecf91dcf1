#!/usr/bin/env python
"""Forced on-device tune of one bench workload (diagnostic): python scripts/tune_one.py ffn"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2210_09603_b200 import tune, workloads as W
    dev = torch.device("cuda", 0)
    rnd = lambda s, dt=torch.bfloat16: torch.empty(s, device=dev).uniform_(-1, 1).to(dt)
    T = W.BERT_TOKENS
    ins = [rnd((T, 768)), rnd((768, 3072)), rnd((3072,)), rnd((3072, 768)), rnd((768,))]
    outs = [torch.empty((T, 768), device=dev, dtype=torch.bfloat16)]
    t0 = time.time()
    best, rep = tune(W.ffn_dag(T), ins, outs)
    print("tuned", best, f"{time.time() - t0:.1f}s", rep["best_ms"], flush=True)


if __name__ == "__main__":
    main()
