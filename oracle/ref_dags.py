"""TEST INFRASTRUCTURE ONLY -- the BASELINE workload DAGs built with the
reference's own builders (proj/src/compute_ir.cpp:496-597 through oracle/_ref)
plus epilogue nodes appended in the DAG JSON wire form, without
touching the product library.  Used by bench.py's cpu_baseline leg and its
reference arm, so that arm runs the unmodified reference end to end:
reference builders -> reference_eval.

Expressions are the JSON prefix lists of the wire form: ["i", n], ["f", x],
["v", axis], ["load", tensor, idx...], [binop, a, b], [unop, a],
["select", c, t, e].
"""
import json
from typing import Sequence

from . import ref_build


def _v(n):
    return ["v", n]


def _load(t, idx):
    return ["load", t, *idx]


def _gelu_tanh(x):
    """tanh-form GELU with Exp/Div (the reference IR has no tanh, proj/include/taskmap/expr.hpp:16)."""
    x3 = ["mul", ["mul", x, x], x]
    inner = ["mul", ["f", 0.7978845608028654], ["add", x, ["mul", ["f", 0.044715], x3]]]
    t = ["sub", ["f", 1.0], ["div", ["f", 2.0], ["add", ["exp", ["mul", ["f", 2.0], inner]], ["f", 1.0]]]]
    return ["mul", ["mul", ["f", 0.5], x], ["add", ["f", 1.0], t]]


def _input(name, shape):
    return {"name": name, "shape": list(shape), "dtype": "f32", "kind": "input"}


def _compute(name, axes, value):
    return {"name": name, "shape": [e for _, e in axes], "dtype": "f32", "kind": "compute",
            "axes": [list(a) for a in axes], "value": value}


def _reduce(name, axes, raxes, value):
    return {"name": name, "shape": [e for _, e in axes], "dtype": "f32", "kind": "reduce",
            "axes": [list(a) for a in axes], "reduce_axes": [list(a) for a in raxes], "combiner": "sum",
            "value": value}


def conv_bn_relu(n: int, c: int, h: int, f: int, k: int, s: int, p: int) -> str:
    """config 3: conv2d_im2col_dag (compute_ir.cpp:517-597) + Z = relu(Out*Scale[p] + Shift[p])."""
    d = json.loads(ref_build("conv2d_im2col", [n, c, h, h, f, k, k, s, p, 0]))
    out = next(x for x in d["nodes"] if x["name"] == "Out")
    d["nodes"] += [_input("Scale", [f]), _input("Shift", [f])]
    d["inputs"] += ["Scale", "Shift"]
    x = _load("Out", [_v("n"), _v("p"), _v("oh"), _v("ow")])
    d["nodes"].append(_compute("Z", out["axes"], ["relu", ["add", ["mul", x, _load("Scale", [_v("p")])],
                                                           _load("Shift", [_v("p")])]]))
    d["outputs"] = ["Z"]
    return json.dumps(d)


def ffn(t: int, dm: int = 768, dff: int = 3072) -> str:
    """config 4: H = gelu_tanh(X W1 + b1); O = H W2 + b2 + X (hand-built, as the probe in SURVEY §8c)."""
    nodes = [_input("X", [t, dm]), _input("W1", [dm, dff]), _input("b1", [dff]), _input("W2", [dff, dm]),
             _input("b2", [dm])]
    nodes.append(_reduce("H0", [("t", t), ("f", dff)], [("k", dm)],
                         ["mul", _load("X", [_v("t"), _v("k")]), _load("W1", [_v("k"), _v("f")])]))
    nodes.append(_compute("H", [("t", t), ("f", dff)],
                          _gelu_tanh(["add", _load("H0", [_v("t"), _v("f")]), _load("b1", [_v("f")])])))
    nodes.append(_reduce("O0", [("t", t), ("d", dm)], [("k", dff)],
                         ["mul", _load("H", [_v("t"), _v("k")]), _load("W2", [_v("k"), _v("d")])]))
    nodes.append(_compute("O", [("t", t), ("d", dm)],
                          ["add", ["add", _load("O0", [_v("t"), _v("d")]), _load("b2", [_v("d")])],
                           _load("X", [_v("t"), _v("d")])]))
    return json.dumps({"nodes": nodes, "inputs": ["X", "W1", "b1", "W2", "b2"], "outputs": ["O"]})


def attention_scores(b: int, s: int = 128, dh: int = 64, scale: float = 0.125) -> str:
    """config 2: S[b,i,j] = scale * sum_k Q[b,i,k] K[b,j,k] (GridReduce with a batch axis)."""
    nodes = [_input("Q", [b, s, dh]), _input("K", [b, s, dh])]
    ax = [("b", b), ("i", s), ("j", s)]
    nodes.append(_reduce("S0", ax, [("k", dh)], ["mul", _load("Q", [_v("b"), _v("i"), _v("k")]),
                                                  _load("K", [_v("b"), _v("j"), _v("k")])]))
    nodes.append(_compute("S", ax, ["mul", _load("S0", [_v("b"), _v("i"), _v("j")]), ["f", scale]]))
    return json.dumps({"nodes": nodes, "inputs": ["Q", "K"], "outputs": ["S"]})


def matmul_bias_relu(m: int, n: int, k: int) -> str:
    """config 1: matmul_dag (compute_ir.cpp:496-515) + D = relu(C + Bias[j])."""
    d = json.loads(ref_build("matmul", [m, n, k, 0]))
    d["nodes"].append(_input("Bias", [n]))
    d["inputs"].append("Bias")
    d["nodes"].append(_compute("D", [("i", m), ("j", n)],
                               ["relu", ["add", _load("C", [_v("i"), _v("j")]), _load("Bias", [_v("j")])]]))
    d["outputs"] = ["D"]
    return json.dumps(d)


def shapes_of(dag_json: str, names: Sequence[str]):
    d = json.loads(dag_json)
    return {x["name"]: tuple(x["shape"]) for x in d["nodes"] if x["name"] in names}
