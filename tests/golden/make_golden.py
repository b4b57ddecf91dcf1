#!/usr/bin/env python
"""Generates the golden fixtures in tests/golden/ from the REAL reference
library (oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile).

The fixtures pin the numpy port (oracle/port.py) and the product's host-side
IR (mapping algebra, builders, classify) on machines where the reference is not
available (the GPU box has no /root/reference).  Re-run after changing the
corpus:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from corpus import classify_corpus, dag_cases, mapping_corpus  # noqa: E402


def main():
    if not oracle.ref_available():
        sys.exit("oracle/_ref/libtaskmap_ref.so missing: run `make -C oracle` first")
    arrays = {}
    meta = {"rng": [], "dags": [], "mappings": [], "classify": [], "builders": {}}
    # splitmix64 streams of taskmap::Rng / random_tensor (tensor.cpp:42-69)
    for seed in (0, 1, 2, 5, 12345):
        f, i = oracle.ref_random_stream(seed, [((257,), False), ((257,), True)])
        arrays[f"rng_f32_{seed}"] = f
        arrays[f"rng_i32_{seed}"] = i
        meta["rng"].append(seed)
    # reference_eval on small instances of every BASELINE config chain
    for name, dag, inputs, outs in dag_cases():
        res = oracle.ref_eval(dag.to_json(), inputs, list(outs), outs)
        for k, v in inputs.items():
            arrays[f"dag_{name}_in_{k}"] = v
        for k, v in res.items():
            arrays[f"dag_{name}_out_{k}"] = v
        meta["dags"].append({"name": name, "dag": dag.to_json(), "inputs": list(inputs), "outputs": list(outs)})
    # task-mapping assignments
    for text in mapping_corpus():
        w, d, t, shape = oracle.ref_mapping_info(text)
        meta["mappings"].append({"text": text, "workers": w, "task_dim": d, "tasks_per_worker": t,
                                 "shape": list(shape), "canonical": oracle.ref_mapping_text(text),
                                 "visualize": oracle.ref_mapping_text(text, True) if d <= 2 and w * t <= 256 else None,
                                 "workers_checked": sorted({0, w // 2, w - 1} | set(range(min(w, 8)))),
                                 "assign": [oracle.ref_mapping_assign(text, k)
                                            for k in sorted({0, w // 2, w - 1} | set(range(min(w, 8))))]})
    # classify decisions
    for name, dag_json, node in classify_corpus():
        meta["classify"].append({"name": name, "dag": dag_json, "node": node,
                                 "class": oracle.ref_classify(dag_json, node)})
    # reference builder output (expression trees), for builder parity
    for kind, args in [("matmul", [3, 4, 5, 0]), ("matmul", [2, 2, 2, 1]),
                       ("conv2d_im2col", [1, 2, 5, 5, 3, 3, 3, 2, 1, 0]),
                       ("conv2d_im2col", [2, 3, 7, 6, 4, 1, 1, 1, 0, 1]),
                       ("batchnorm", [2, 3, 4, 4, 0]), ("transpose", [0, 3, 2, 3, 4, 2, 0, 1]),
                       ("reshape", [0, 1, 100, 2, 2, 50]), ("reshape", [0, 2, 2, 50, 1, 100])]:
        meta["builders"][f"{kind}:{','.join(map(str, args))}"] = oracle.ref_build(kind, args)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(meta['dags'])} DAG cases, {len(meta['mappings'])} mappings, "
          f"{len(meta['classify'])} classify cases")


if __name__ == "__main__":
    main()
