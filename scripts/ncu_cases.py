#!/usr/bin/env python
"""Extra single-workload launchers for ncu captures (profiles/): the config-1
fp32 CUDA-core and tf32 kernels and the rule-based / reduce-template kernels.
  python scripts/ncu_cases.py simt|tf32|softmax [--iters N]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2210_09603_b200 import (Axis, ComputeDAG, DType, Plan, ScheduleConfig, TensorNode, div, exp, load,
                                       sub, var, workloads as W)
    from paper_2210_09603_b200 import taskmap as T
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    r = lambda *s: torch.empty(s, device=dev).uniform_(-1, 1)  # noqa: E731
    if a.case in ("simt", "tf32"):
        m = n = k = 1024
        ins, outs = [r(m, k), r(k, n), r(n)], [torch.empty((m, n), device=dev)]
        cfg = ScheduleConfig(math="fp32_simt", block_n=64) if a.case == "simt" else ScheduleConfig(math="tf32")
        ex = Plan(W.matmul_bias_relu_dag(m, n, k), cfg).bind(ins, outs)
    else:  # row softmax over 8192 x 3072 (the BERT FFN width): max / exp / sum / div
        rows, cols = 8192, 3072
        d = ComputeDAG()
        d.add_input("X", [rows, cols])
        i, j, kk = var("i"), var("j"), var("k")
        d.nodes.append(TensorNode("M", [rows], DType.F32, "reduce", [Axis("i", rows)], [Axis("k", cols)],
                                  combiner=T.Combiner.Max, value=load("X", [i, kk])))
        d.add_compute("E", [Axis("i", rows), Axis("j", cols)], exp(sub(load("X", [i, j]), load("M", [i]))))
        d.nodes.append(TensorNode("Z", [rows], DType.F32, "reduce", [Axis("i", rows)], [Axis("k", cols)],
                                  value=load("E", [i, kk])))
        d.add_compute("P", [Axis("i", rows), Axis("j", cols)], div(load("E", [i, j]), load("Z", [i])))
        d.outputs = ["P"]
        ex = Plan(d).bind([r(rows, cols).to(torch.bfloat16)], [torch.empty((rows, cols), device=dev,
                                                                            dtype=torch.bfloat16)])
    for _ in range(a.iters):
        ex.launch()
    torch.cuda.synchronize()
    print(ex.kernel_info(0))


if __name__ == "__main__":
    main()
