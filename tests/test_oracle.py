"""Pins the oracle before trusting it (CPU-only).

* oracle/_ref (the real reference library) reproduces the SPEC's known answers;
* the numpy port (oracle/port.py) equals reference_eval on every golden DAG
  case and reproduces the reference's splitmix64 streams bit for bit;
* when oracle/_ref is present, the golden fixtures are re-derived live.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import port

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")


@pytest.mark.parametrize("seed", META["rng"])
def test_port_rng_matches_reference_stream(seed):
    """splitmix64 Rng + random_tensor (tensor.cpp:42-69): f32 -> U(-1,1), i32 -> U{-8..8}."""
    r = port.Rng(seed)
    assert np.array_equal(r.tensor((257,)), GOLD[f"rng_f32_{seed}"])
    assert np.array_equal(r.tensor((257,), True), GOLD[f"rng_i32_{seed}"])


def _port_eval(name, ins):
    if name.startswith("matmul_bias_relu"):
        return {"D": port.matmul_bias_relu(ins["A"], ins["B"], ins["Bias"])}
    if name == "matmul_bias_gelu":
        return {"D": port.gelu_tanh(port.matmul(ins["A"], ins["B"]) + ins["Bias"][None, :])}
    if name == "batched_scale":
        return {"P": port.batched_matmul_scale(ins["Q"], ins["KT"], 0.125)}
    if name.startswith("conv_bn_relu"):
        g = list(map(int, name.split("_")[3:]))
        return {"Z": port.conv_bn_relu(ins["X"], ins["W"], ins["Scale"], ins["Shift"], g[7], g[8])}
    if name == "im2col_col":
        return {"Col": port.im2col(ins["X"], 3, 3, 2, 1), "Out": port.conv2d_nchw(ins["X"], ins["W"], 2, 1)}
    if name == "ffn":
        return {"O": port.ffn(ins["X"], ins["W1"], ins["b1"], ins["W2"], ins["b2"])}
    raise KeyError(name)


@pytest.mark.parametrize("case", [d["name"] for d in META["dags"]])
def test_port_matches_golden_reference_eval(case):
    d = next(x for x in META["dags"] if x["name"] == case)
    ins = {k: GOLD[f"dag_{case}_in_{k}"] for k in d["inputs"]}
    got = _port_eval(case, ins)
    for o in d["outputs"]:
        want = GOLD[f"dag_{case}_out_{o}"]
        if case.endswith("i32") or case == "im2col_col" and o == "Col":
            assert np.array_equal(got[o], want)   # integer / pure-copy work: bit-exact
        else:
            assert port.max_rel_error(got[o], want) <= 1e-12


@needs_ref
def test_reference_spec_known_answers():
    """SPEC.md examples reproduced by the reference library itself."""
    from paper_2210_09603_b200 import Axis, ComputeDAG, DType, TensorNode, conv2d_im2col_dag, load, matmul_dag, var
    d = matmul_dag(2, 2, 2, DType.I32)
    r = oracle.ref_eval(d.to_json(), {"A": np.array([[1, 2], [3, 4]]), "B": np.array([[5, 6], [7, 8]])}, ["C"],
                        {"C": (2, 2)})
    assert r["C"].tolist() == [[19, 22], [43, 50]]
    d = conv2d_im2col_dag(1, 1, 3, 3, 1, 2, 2, 1, 0)
    r = oracle.ref_eval(d.to_json(), {"X": np.ones((1, 1, 3, 3)), "W": np.ones((1, 1, 2, 2))}, ["Out"],
                        {"Out": (1, 1, 2, 2)})
    assert np.all(r["Out"] == 4.0)
    d = ComputeDAG([TensorNode("X", [2039]),  # reduce-sum of 2039 ones
                    TensorNode("Y", [1], kind="reduce", axes=[Axis("i", 1)], reduce_axes=[Axis("r", 2039)],
                               value=load("X", [var("r")]))], ["X"], ["Y"])
    r = oracle.ref_eval(d.to_json(), {"X": np.ones(2039)}, ["Y"], {"Y": (1,)})
    assert r["Y"][0] == 2039.0


@needs_ref
def test_golden_fixtures_rederived_live():
    """The committed fixtures are exactly what the reference computes now."""
    for d in META["dags"][:6]:
        ins = {k: GOLD[f"dag_{d['name']}_in_{k}"] for k in d["inputs"]}
        shapes = {o: GOLD[f"dag_{d['name']}_out_{o}"].shape for o in d["outputs"]}
        res = oracle.ref_eval(d["dag"], ins, d["outputs"], shapes)
        for o in d["outputs"]:
            assert np.array_equal(res[o], GOLD[f"dag_{d['name']}_out_{o}"])
    for seed in META["rng"]:
        f, i = oracle.ref_random_stream(seed, [((257,), False), ((257,), True)])
        assert np.array_equal(f, GOLD[f"rng_f32_{seed}"]) and np.array_equal(i, GOLD[f"rng_i32_{seed}"])


@needs_ref
def test_fold_batchnorm_matches_reference():
    r = port.Rng(9)
    g, b, m, v = r.tensor((7,)) + 1.5, r.tensor((7,)), r.tensor((7,)), r.tensor((7,)) + 1.5
    s_ref, t_ref = oracle.ref_fold_bn(g, b, m, v, 1e-5)
    s, t = port.fold_batchnorm_params(g, b, m, v, 1e-5)
    assert np.array_equal(s, s_ref) and np.array_equal(t, t_ref)


def test_max_rel_error_metric():
    """tensor.cpp:71-86: absolute below 1, relative above (1e-4 example)."""
    assert abs(port.max_rel_error([0.5, 100, -3], [0.5001, 100.01, -3]) - 1e-4) < 1e-12


def test_round_bf16_tf32():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 2 ** -7 + 2 ** -9, -3.14159, 65504.0])
    assert port.round_bf16(x)[0] == 1.0
    assert port.round_bf16(x)[1] == 1.0          # tie -> even
    assert port.round_tf32(np.array([1.0 + 2 ** -11]))[0] == 1.0
    assert np.all(np.abs(port.round_bf16(x) - x) <= np.abs(x) * 2 ** -8)
