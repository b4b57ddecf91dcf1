"""The tuner's correctness gate and the device DAG interpreter
behind it (tm_dag_eval).

* tm_dag_eval is pinned to the reference's reference_eval (oracle/_ref): bit-exact
  on the reference's integer test data, fp64-close on float data.
* tm_tune verifies every schedule against it on seeded inputs and is a hard
  gate: a correct space tunes with zero incorrect configs; broken tensor
  programs (fault injection TMB_FAULT_SKIP_KBLOCK drops each kernel's last
  k-block) abort tuning with status 1 (TM_ERR_CORRECTNESS) and a report.
"""
import os

import numpy as np
import pytest

from oracle import port
from paper_2210_09603_b200 import DType, ScheduleConfig, TaskmapError, dag_eval, schedule_space, tune

from dags import batched_matmul_scale_dag, conv_bn_relu_dag, ffn_dag, matmul_epilogue_dag
from gpu_util import dev, have_ref, oracle_eval

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _eval(dag, inputs_np, dtypes, out_shapes, layouts=None):
    t = _torch()
    layouts = layouts or {}
    ins = [dev(inputs_np[n], dtypes.get(n, "f32"), layouts.get(n)) for n in dag.inputs]
    outs = [t.full(tuple(out_shapes[o]), float("nan"), dtype=t.float32, device="cuda") for o in dag.outputs]
    dag_eval(dag, ins, outs)
    t.cuda.synchronize()
    return {o: x.cpu().numpy().astype(np.float64) for o, x in zip(dag.outputs, outs)}


def _need_ref():
    if not have_ref():
        pytest.skip("reference library (oracle/_ref) not built")


@pytest.mark.parametrize("layout", [None, "cl"])
def test_dag_eval_conv_equals_reference_eval(layout):
    """im2col conv + BN-fold + ReLU (select / floor div-mod index math) on i32 data, any input strides."""
    _need_ref()
    n, c, h, w, f, k, s, p = 2, 5, 7, 9, 6, 3, 2, 1
    rng = port.Rng(71)
    ins = {"X": rng.tensor((n, c, h, w), True), "W": rng.tensor((f, c, k, k), True),
           "Scale": rng.tensor((f,), True), "Shift": rng.tensor((f,), True)}
    dag = conv_bn_relu_dag(n, c, h, w, f, k, k, s, p, DType.I32)
    ho, wo = port.conv_out_extent(h, k, s, p), port.conv_out_extent(w, k, s, p)
    got = _eval(dag, ins, {"X": "bf16", "W": "bf16"}, {"Z": (n, f, ho, wo)}, {"X": layout, "W": layout})
    want = oracle_eval(dag, ins, {"Z": (n, f, ho, wo)})
    assert np.array_equal(got["Z"], want["Z"])


def test_dag_eval_batched_and_matmul_equal_reference_eval():
    _need_ref()
    rng = port.Rng(72)
    q, kt = rng.tensor((3, 16, 8), True), rng.tensor((3, 8, 12), True)
    dag = batched_matmul_scale_dag(3, 16, 12, 8, 0.125, DType.F32)
    got = _eval(dag, {"Q": q, "KT": kt}, {}, {"P": (3, 16, 12)})
    assert np.array_equal(got["P"], oracle_eval(dag, {"Q": q, "KT": kt}, {"P": (3, 16, 12)})["P"])
    a, b, bias = rng.tensor((33, 17), True), rng.tensor((17, 29), True), rng.tensor((29,), True)
    dag = matmul_epilogue_dag(33, 29, 17, DType.I32)
    got = _eval(dag, {"A": a, "B": b, "Bias": bias}, {"A": "bf16"}, {"D": (33, 29)}, {"B": "t"})
    assert np.array_equal(got["D"], oracle_eval(dag, {"A": a, "B": b, "Bias": bias}, {"D": (33, 29)})["D"])


def test_dag_eval_ffn_float_close_to_reference_eval():
    """Float data with exp/div (tanh-form GELU): fp64 on both sides."""
    _need_ref()
    rng = port.Rng(73)
    t, dm, dff = 4, 16, 24
    ins = {"X": rng.tensor((t, dm)), "W1": rng.tensor((dm, dff)), "b1": rng.tensor((dff,)),
           "W2": rng.tensor((dff, dm)), "b2": rng.tensor((dm,))}
    ins = {k: port.round_bf16(v) for k, v in ins.items()}  # exact in f32 storage
    dag = ffn_dag(t, dm, dff)
    got = _eval(dag, ins, {}, {"O": (t, dm)})
    want = oracle_eval(dag, ins, {"O": (t, dm)})["O"]
    assert np.abs(got["O"] - np.asarray(want, np.float32)).max() <= 1e-5 * np.abs(want).max()


def test_dag_eval_reduce_combiners_and_int_index_math():
    """Max/Min combiners from their identities, floor div/mod of negative values, select."""
    _need_ref()
    from paper_2210_09603_b200 import Axis, ComputeDAG, TensorNode, load, var, select, lt, imm, div, mod, sub, add
    from paper_2210_09603_b200.taskmap import Combiner
    d = ComputeDAG()
    d.add_input("X", [5, 7], DType.I32)
    for name, comb in (("Mx", Combiner.Max), ("Mn", Combiner.Min)):
        d.nodes.append(TensorNode(name, [5], DType.I32, "reduce", [Axis("i", 5)], [Axis("j", 7)], comb,
                                  load("X", [var("i"), var("j")])))
    x = load("X", [var("i"), var("j")])
    d.add_compute("Q", [Axis("i", 5), Axis("j", 7)],
                  add(add(div(x, imm(3)), mod(x, imm(4))),
                      select(lt(x, imm(0)), load("Mx", [var("i")]), sub(imm(0), load("Mn", [var("i")])))), DType.I32)
    d.outputs = ["Mx", "Mn", "Q"]
    xv = port.Rng(74).tensor((5, 7), True)
    shapes = {"Mx": (5,), "Mn": (5,), "Q": (5, 7)}
    got = _eval(d, {"X": xv}, {}, shapes)
    want = oracle_eval(d, {"X": xv}, shapes)
    for o in shapes:
        assert np.array_equal(got[o], want[o]), o


def _ffn_tensors(t, dm, dff, seed=5):
    torch = _torch()
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    r = lambda *s: torch.empty(s, device="cuda").uniform_(-1, 1, generator=g).to(torch.bfloat16)
    ins = [r(t, dm), r(dm, dff), r(dff), r(dff, dm), r(dm)]
    outs = [torch.empty((t, dm), device="cuda", dtype=torch.bfloat16)]
    return ins, outs


def test_tune_ffn_chain_every_config_correct():
    """The FFN chain (GELU GEMM -> residual GEMM), where round 1's gate rejected every
    split-K schedule: with a scale-aware float gate and the integer trial, every
    config of the space (split-K 1/2/4, pairs, half grids) must pass."""
    t, dm, dff = 512, 256, 1024
    ins, outs = _ffn_tensors(t, dm, dff)
    best, rep = tune(ffn_dag(t, dm, dff), ins, outs, reps=2)
    assert rep["ok"] and rep["n_incorrect"] == 0
    assert rep["space_size"] == len(schedule_space("matmul"))
    assert rep["n_correct"] + rep["n_unsupported"] == rep["space_size"]
    assert rep["n_correct"] >= rep["space_size"] - 4
    assert best in schedule_space("matmul")
    assert not rep["verification"]["integer_exact"]  # exp/div in GELU: float gate on both trials


def test_tune_conv_integer_trial_is_bit_exact():
    torch = _torch()
    n, c, h, f, k, s, p = 2, 64, 14, 128, 3, 1, 1
    dag = conv_bn_relu_dag(n, c, h, h, f, k, k, s, p)
    cl = torch.channels_last
    ins = [torch.randn(n, c, h, h, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl),
           torch.randn(f, c, k, k, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl),
           torch.rand(f, device="cuda"), torch.randn(f, device="cuda")]
    outs = [torch.empty(n, f, h, h, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)]
    _, rep = tune(dag, ins, outs, reps=2)
    assert rep["ok"] and rep["verification"]["integer_exact"]
    for r in rep["results"]:
        if r["status"] == "correct":
            assert r["int_mismatches"] == 0


def test_tune_gate_aborts_on_incorrect_configs(monkeypatch):
    """Tensor programs that drop their last k-block (fault injection TMB_FAULT_SKIP_KBLOCK) must
    abort tuning with TM_ERR_CORRECTNESS and a report, not be skipped."""
    t, dm, dff = 256, 128, 256
    ins, outs = _ffn_tensors(t, dm, dff)
    monkeypatch.setenv("TMB_FAULT_SKIP_KBLOCK", "1")
    with pytest.raises(TaskmapError) as e:
        tune(ffn_dag(t, dm, dff), ins, outs, reps=1)
    assert e.value.status == 1
    rep = e.value.report
    assert rep is not None and not rep["ok"] and rep["n_incorrect"] > 0 and rep["n_correct"] == 0
