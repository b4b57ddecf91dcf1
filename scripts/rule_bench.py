"""Rule-based / reduce kernels: the NVRTC-generated kernels
against the bytecode interpreter on HBM-sized inputs, as HBM bandwidth.
Usage (GPU box): python scripts/rule_bench.py > gpurun_out/rule_bench.json"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2210_09603_b200 import (Axis, ComputeDAG, DType, Plan, ScheduleConfig, TensorNode, div, exp, load,  # noqa: E402
                                   relu, sub, var)
from paper_2210_09603_b200 import taskmap as T  # noqa: E402


def relu_dag(n):
    d = ComputeDAG()
    d.add_input("X", [n])
    d.add_compute("Y", [Axis("i", n)], relu(load("X", [var("i")])))
    d.outputs = ["Y"]
    return d, {"X": (n,)}, {"Y": (n,)}, 8 * n


def softmax_dag(rows, cols):
    d = ComputeDAG()
    d.add_input("X", [rows, cols])
    i, j, k = var("i"), var("j"), var("k")
    d.nodes.append(TensorNode("M", [rows], DType.F32, "reduce", [Axis("i", rows)], [Axis("k", cols)],
                              combiner=T.Combiner.Max, value=load("X", [i, k])))
    d.add_compute("E", [Axis("i", rows), Axis("j", cols)], exp(sub(load("X", [i, j]), load("M", [i]))))
    d.nodes.append(TensorNode("Z", [rows], DType.F32, "reduce", [Axis("i", rows)], [Axis("k", cols)],
                              value=load("E", [i, k])))
    d.add_compute("P", [Axis("i", rows), Axis("j", cols)], div(load("E", [i, j]), load("Z", [i])))
    d.outputs = ["P"]
    # algorithmic bytes: read X (max), read X + write E, read E (sum), read E + write P
    return d, {"X": (rows, cols)}, {"P": (rows, cols)}, 4 * rows * cols * 6


def rowsum_dag(rows, cols):
    d = ComputeDAG()
    d.add_input("X", [rows, cols])
    d.nodes.append(TensorNode("S", [rows], DType.F32, "reduce", [Axis("i", rows)], [Axis("k", cols)],
                              value=load("X", [var("i"), var("k")])))
    d.outputs = ["S"]
    return d, {"X": (rows, cols)}, {"S": (rows,)}, 4 * rows * cols


def time_exec(ex, iters=20):
    s = torch.cuda.current_stream()
    for _ in range(3):
        ex.launch(s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(iters):
        ex.launch(s)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    cases = [("relu_64M", relu_dag(1 << 26)), ("softmax_8192x4096", softmax_dag(8192, 4096)),
             ("rowsum_16x4M", rowsum_dag(16, 1 << 22)), ("rowsum_1Mx32", rowsum_dag(1 << 20, 32))]
    out = []
    for name, (dag, ins, outs, algo_bytes) in cases:
        xs = [torch.randn(ins[n], device="cuda") for n in dag.inputs]
        ys = [torch.empty(outs[o], device="cuda") for o in dag.outputs]
        row = {"case": name, "algorithmic_bytes": algo_bytes}
        res = {}
        for mode in ("generated", "interpreter"):
            if mode == "interpreter":
                os.environ["TMB_RULE_INTERP"] = "1"
            else:
                os.environ.pop("TMB_RULE_INTERP", None)
            ex = Plan(dag, ScheduleConfig(threads_per_block=256)).bind(xs, ys)
            ms = time_exec(ex)
            torch.cuda.synchronize()
            res[mode] = ys[0].clone()
            row[mode] = {"ms": round(ms, 4), "GB/s": round(algo_bytes / ms / 1e6, 1),
                         "kinds": [ex.kernel_kind(i) for i in range(ex.num_launches)]}
        row["bit_identical"] = bool(torch.equal(res["generated"].view(torch.int32), res["interpreter"].view(torch.int32)))
        out.append(row)
        print(json.dumps(row), flush=True)
    os.environ.pop("TMB_RULE_INTERP", None)


if __name__ == "__main__":
    main()
