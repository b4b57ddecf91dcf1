"""Rule-based injective kernels and the reduce template (SPEC.md:282-290,
:300-308), and partition over multi-anchor graphs with
anchor-free subgraphs (row f4), checked against the reference's reference_eval
(oracle/_ref) on the same inputs: exact on the reference's integer data,
max_rel_error <= 1e-5 on fp32 data (fp32 device arithmetic vs the fp64 oracle).
"""
import numpy as np
import pytest

from gpu_util import dev, have_ref, oracle_eval, run
from oracle import port
from paper_2210_09603_b200 import (Axis, ComputeDAG, DType, Plan, ScheduleConfig, TensorNode, add, div, exp, fimm,
                                   load, maximum, mul, relu, sub, var)
from paper_2210_09603_b200 import taskmap as T

pytestmark = pytest.mark.gpu


def _need_ref():
    if not have_ref():
        pytest.skip("reference library (oracle/_ref) not built")


def _check(dag, inputs_np, out_shapes, exact, cfg=None, dtype="f32"):
    _need_ref()
    got, plan = run(dag, {k: dev(v, dtype) for k, v in inputs_np.items()}, out_shapes, "f32", cfg)
    want = oracle_eval(dag, inputs_np, out_shapes)
    for o in dag.outputs:
        if exact:
            assert np.array_equal(got[o], want[o]), o
        else:
            assert port.max_rel_error(got[o], want[o]) <= 1e-5, (o, port.max_rel_error(got[o], want[o]))
    return plan


def test_relu_1000_elements_rule_kernel():
    """ReLU on 1000 elements -> one rule-based kernel, guard idx < 1000."""
    d = ComputeDAG()
    d.add_input("X", [1000], DType.I32)
    d.add_compute("Y", [Axis("i", 1000)], relu(load("X", [var("i")])), DType.I32)
    d.outputs = ["Y"]
    plan = _check(d, {"X": port.Rng(501).tensor((1000,), True)}, {"Y": (1000,)}, exact=True)
    assert [k["kind"] for k in plan.describe()["kernels"]] == ["rule"]


def test_reshape_only_dag_is_a_copy():
    """a reshape-only DAG is a pure copy equal to the reference."""
    d = T.reshape_dag([6, 35], [2, 3, 5, 7], DType.I32)
    x = port.Rng(502).tensor((6, 35), True)
    name_in, name_out = d.inputs[0], d.outputs[0]
    _check(d, {name_in: x}, {name_out: (2, 3, 5, 7)}, exact=True)


def test_elementwise_chain_fused_in_one_kernel():
    """a*2+1 fused into one store, equal to the oracle."""
    d = ComputeDAG()
    d.add_input("A", [37, 41], DType.I32)
    ax = [Axis("i", 37), Axis("j", 41)]
    d.add_compute("T1", ax, mul(load("A", [var("i"), var("j")]), T.imm(2)), DType.I32)
    d.add_compute("T2", ax, add(load("T1", [var("i"), var("j")]), T.imm(1)), DType.I32)
    d.outputs = ["T2"]
    plan = _check(d, {"A": port.Rng(503).tensor((37, 41), True)}, {"T2": (37, 41)}, exact=True)
    (k,) = plan.describe()["kernels"]
    assert k["kind"] == "rule" and k["inlined"] == ["T1"]


@pytest.mark.parametrize("n,threads", [(2048, 128), (1, 128), (2039, 256), (100000, 512)])
def test_reduce_template_sums(n, threads):
    """sum of 2048 ones with 128 threads = 2048; a single element;
    the prime extent 2039 (guarded tail); a long reduction over 512 threads."""
    d = ComputeDAG()
    d.add_input("X", [n], DType.I32)
    d.nodes.append(TensorNode("S", [1], DType.I32, "reduce", [Axis("o", 1)], [Axis("k", n)],
                              value=load("X", [var("k")])))
    d.outputs = ["S"]
    x = np.ones(n) if n == 2048 else port.Rng(504 + n).tensor((n,), True)
    got, plan = run(d, {"X": dev(x, "f32")}, {"S": (1,)}, "f32", ScheduleConfig(threads_per_block=threads))
    assert got["S"][0] == x.sum()
    assert plan.describe()["kernels"][0]["kind"] == "reduce"


def test_max_of_single_element():
    d = ComputeDAG()
    d.add_input("X", [1])
    d.nodes.append(TensorNode("M", [1], DType.F32, "reduce", [Axis("o", 1)], [Axis("k", 1)],
                              combiner=T.Combiner.Max, value=load("X", [var("k")])))
    d.outputs = ["M"]
    got, _ = run(d, {"X": dev(np.array([-3.25]), "f32")}, {"M": (1,)})
    assert got["M"][0] == -3.25


def _softmax_dag(rows, cols):
    """Row softmax as the reference's IR writes it: a max reduction, exp, a sum
    reduction, a division -- two non-matmul reductions and two injective nodes."""
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
    return d


@pytest.mark.parametrize("rows,cols", [(64, 200), (3, 4099), (1000, 7)])
def test_softmax_graph(rows, cols):
    d = _softmax_dag(rows, cols)
    plan = _check(d, {"X": port.Rng(505).tensor((rows, cols)) * 4.0}, {"P": (rows, cols)}, exact=False)
    kinds = [(k["kind"], k["root"]) for k in plan.describe()["kernels"]]
    assert kinds == [("reduce", "M"), ("rule", "E"), ("reduce", "Z"), ("rule", "P")], kinds


def test_global_average_pool_and_2x2_pool():
    """Pooling as reductions: a 7x7 global average (sum, then x 1/49) and a 2x2
    stride-2 max pool (reduce extent 4: the in-thread sequential loop)."""
    n, c, h = 2, 16, 14
    d = ComputeDAG()
    d.add_input("X", [n, c, h, h], DType.I32)
    nn, cc, y, x, r, s = var("n"), var("c"), var("y"), var("x"), var("r"), var("s")
    d.nodes.append(TensorNode("MP", [n, c, h // 2, h // 2], DType.I32, "reduce",
                              [Axis("n", n), Axis("c", c), Axis("y", h // 2), Axis("x", h // 2)],
                              [Axis("r", 2), Axis("s", 2)], combiner=T.Combiner.Max,
                              value=load("X", [nn, cc, add(mul(y, T.imm(2)), r), add(mul(x, T.imm(2)), s)])))
    d.nodes.append(TensorNode("GS", [n, c], DType.I32, "reduce", [Axis("n", n), Axis("c", c)],
                              [Axis("r", h // 2), Axis("s", h // 2)], value=load("MP", [nn, cc, r, s])))
    d.outputs = ["MP", "GS"]
    xv = port.Rng(506).tensor((n, c, h, h), True)
    _check(d, {"X": xv}, {"MP": (n, c, h // 2, h // 2), "GS": (n, c)}, exact=True)


def _attention_dag(b, s, dh, scale):
    """S = scale * Q K^T (GEMM + epilogue), P = softmax(S) (reduce / rule kernels),
    O = P V (GEMM whose prologue P reads intermediates: materialised first)."""
    d = ComputeDAG()
    d.add_input("Q", [b, s, dh])
    d.add_input("Kt", [b, s, dh])
    d.add_input("V", [b, s, dh])
    bb, i, j, k = var("b"), var("i"), var("j"), var("k")
    ax3 = [Axis("b", b), Axis("i", s), Axis("j", s)]
    d.nodes.append(TensorNode("S0", [b, s, s], DType.F32, "reduce", ax3, [Axis("k", dh)],
                              value=mul(load("Q", [bb, i, k]), load("Kt", [bb, j, k]))))
    d.add_compute("S", ax3, mul(load("S0", [bb, i, j]), fimm(scale)))
    d.nodes.append(TensorNode("M", [b, s], DType.F32, "reduce", [Axis("b", b), Axis("i", s)], [Axis("k", s)],
                              combiner=T.Combiner.Max, value=load("S", [bb, i, k])))
    d.add_compute("E", ax3, exp(sub(load("S", [bb, i, j]), load("M", [bb, i]))))
    d.nodes.append(TensorNode("Z", [b, s], DType.F32, "reduce", [Axis("b", b), Axis("i", s)], [Axis("k", s)],
                              value=load("E", [bb, i, k])))
    d.add_compute("P", ax3, div(load("E", [bb, i, j]), load("Z", [bb, i])))
    d.nodes.append(TensorNode("O", [b, s, dh], DType.F32, "reduce", [Axis("b", b), Axis("i", s), Axis("d", dh)],
                              [Axis("k", s)], value=mul(load("P", [bb, i, k]), load("V", [bb, k, var("d")]))))
    d.outputs = ["O"]
    return d


def test_attention_graph_partition_and_parity():
    """Row f4: partition of a multi-anchor graph (two matmul anchors, two
    non-matmul reductions, anchor-free exp/div) into tcgen05 GEMMs, reduce-template
    and rule-based kernels; the whole graph equals reference_eval."""
    b, s, dh = 2, 128, 64
    d = _attention_dag(b, s, dh, 0.125)
    rng = port.Rng(507)
    q, kt, v = (rng.tensor((b, s, dh)) for _ in range(3))
    # fp32 inputs: math auto runs both GEMMs on the exact-fp32 CUDA-core template
    plan = _check(d, {"Q": q, "Kt": kt, "V": v}, {"O": (b, s, dh)}, exact=False)
    kinds = [(k["kind"], k.get("root", k.get("anchor"))) for k in plan.describe()["kernels"]]
    assert kinds == [("gemm", "S0"), ("reduce", "M"), ("rule", "E"), ("reduce", "Z"), ("rule", "P"),
                     ("gemm", "O")], kinds


def test_epilogue_beyond_the_register_program_is_cut_into_a_rule_kernel():
    """A GEMM epilogue using an op the register program lacks (max against a
    tensor element read twice) is cut: the GEMM keeps what lowers, a rule kernel
    runs the rest."""
    m, n, k = 128, 96, 64
    d = ComputeDAG()
    d.add_input("A", [m, k], DType.I32)
    d.add_input("B", [k, n], DType.I32)
    i, j, kk = var("i"), var("j"), var("k")
    d.nodes.append(TensorNode("C", [m, n], DType.I32, "reduce", [Axis("i", m), Axis("j", n)], [Axis("k", k)],
                              value=mul(load("A", [i, kk]), load("B", [kk, j]))))
    d.add_compute("D", [Axis("i", m), Axis("j", n)], relu(load("C", [i, j])), DType.I32)
    d.add_compute("F", [Axis("i", m), Axis("j", n)], maximum(load("D", [i, j]), mul(load("D", [i, j]), load("D", [i, j]))),
                  DType.I32)
    d.outputs = ["F"]
    rng = port.Rng(508)
    plan = _check(d, {"A": rng.tensor((m, k), True), "B": rng.tensor((k, n), True)}, {"F": (m, n)}, exact=True)
    assert [k["kind"] for k in plan.describe()["kernels"]] == ["gemm", "rule"]


def _bind_run(dag, inputs, out_shapes, cfg=None):
    import torch
    outs = {o: torch.full(tuple(out_shapes[o]), float("nan"), dtype=torch.float32, device="cuda") for o in dag.outputs}
    plan = Plan(dag, cfg or ScheduleConfig())
    ex = plan.bind([inputs[n] for n in dag.inputs], [outs[o] for o in dag.outputs])
    ex.launch()
    torch.cuda.synchronize()
    kinds = [ex.kernel_kind(i) for i in range(len(plan.describe()["kernels"]))]
    return {o: outs[o].cpu().numpy() for o in dag.outputs}, kinds


def _generated_vs_interpreter(monkeypatch, dag, inputs_np, out_shapes, cfg=None, bitwise=True):
    """The NVRTC-generated rule kernels against the bytecode interpreter: same
    promotion rules, no FMA contraction, same reduction order -> bit-identical."""
    inputs = {k: dev(v, "f32") for k, v in inputs_np.items()}
    monkeypatch.delenv("TMB_RULE_INTERP", raising=False)
    gen, kinds_gen = _bind_run(dag, inputs, out_shapes, cfg)
    monkeypatch.setenv("TMB_RULE_INTERP", "1")
    ref, kinds_ref = _bind_run(dag, inputs, out_shapes, cfg)
    monkeypatch.delenv("TMB_RULE_INTERP")
    for o in dag.outputs:
        if bitwise:
            assert np.array_equal(gen[o].view(np.uint32), ref[o].view(np.uint32)), o
        else:
            assert port.max_rel_error(gen[o], ref[o]) <= 1e-5, o
    assert "rule-interp" not in kinds_gen, kinds_gen
    assert "rule-generated" not in kinds_ref, kinds_ref
    return kinds_gen


def test_generated_softmax_equals_interpreter(monkeypatch):
    kinds = _generated_vs_interpreter(monkeypatch, _softmax_dag(200, 301),
                                      {"X": port.Rng(520).tensor((200, 301)) * 4.0}, {"P": (200, 301)})
    assert kinds == ["rule-generated"] * 4


def _row_reduce_dag(rows, n, dtype, combiner=None):
    d = ComputeDAG()
    d.add_input("X", [rows, n], dtype)
    kw = {} if combiner is None else {"combiner": combiner}
    d.nodes.append(TensorNode("S", [rows], dtype, "reduce", [Axis("o", rows)], [Axis("k", n)],
                              value=mul(load("X", [var("o"), var("k")]), T.imm(3)), **kw))
    d.outputs = ["S"]
    return d


@pytest.mark.parametrize("threads", [64, 128, 256, 512])
@pytest.mark.parametrize("rows,n", [(3, 70001), (1, 1 << 20), (200, 3000), (5000, 48), (777, 17), (20000, 9)])
def test_generated_reduction_shapes(monkeypatch, threads, rows, n):
    """Every generated reduction shape -- SPLIT (fewer outputs than SMs, long
    rows), TREE, GROUP (short rows, many outputs) -- on integer data: int64
    accumulation makes any association exact, so the generated kernels equal the
    interpreter bit for bit; Max is order-free on float data as well."""
    rng = port.Rng(521 + rows)
    x = rng.tensor((rows, n), True)
    d = _row_reduce_dag(rows, n, DType.I32)
    _generated_vs_interpreter(monkeypatch, d, {"X": x}, {"S": (rows,)}, ScheduleConfig(threads_per_block=threads))
    d = _row_reduce_dag(rows, n, DType.F32, T.Combiner.Max)
    _generated_vs_interpreter(monkeypatch, d, {"X": rng.tensor((rows, n))}, {"S": (rows,)},
                              ScheduleConfig(threads_per_block=threads))


@pytest.mark.parametrize("rows,n", [(3, 70001), (5000, 48)])
def test_generated_float_sums_against_the_oracle(rows, n):
    """Float sums under SPLIT / GROUP associate differently from the interpreter:
    checked against reference_eval (fp64) with the fp32 tolerance."""
    d = _row_reduce_dag(rows, n, DType.F32)
    _check(d, {"X": port.Rng(530 + rows).tensor((rows, n))}, {"S": (rows,)}, exact=False)


def test_generated_pooling_integer_and_guards(monkeypatch):
    """Integer max pool + sum with a padding guard (select on bounds), floor
    division / modulo in the indices: the integer semantics of the generated code."""
    n, c, h = 2, 8, 15
    d = ComputeDAG()
    d.add_input("X", [n, c, h, h], DType.I32)
    nn, cc, y, x, r, s = var("n"), var("c"), var("y"), var("x"), var("r"), var("s")
    ho = (h + 1) // 2
    iy, ix = sub(add(mul(y, T.imm(2)), r), T.imm(1)), sub(add(mul(x, T.imm(2)), s), T.imm(1))
    inb = T.land(T.land(T.ge(iy, T.imm(0)), T.lt(iy, T.imm(h))), T.land(T.ge(ix, T.imm(0)), T.lt(ix, T.imm(h))))
    d.nodes.append(TensorNode("MP", [n, c, ho, ho], DType.I32, "reduce",
                              [Axis("n", n), Axis("c", c), Axis("y", ho), Axis("x", ho)],
                              [Axis("r", 3), Axis("s", 3)], combiner=T.Combiner.Max,
                              value=T.select(inb, load("X", [nn, cc, iy, ix]), T.imm(-1000))))
    d.add_compute("Q", [Axis("n", n), Axis("c", c), Axis("y", ho), Axis("x", ho)],
                  add(T.div(load("MP", [nn, cc, y, x]), T.imm(3)), T.mod(load("MP", [nn, cc, y, x]), T.imm(5))),
                  DType.I32)
    d.outputs = ["Q"]
    xv = port.Rng(522).tensor((n, c, h, h), True)
    kinds = _generated_vs_interpreter(monkeypatch, d, {"X": xv}, {"Q": (n, c, ho, ho)})
    assert kinds == ["rule-generated", "rule-generated"]
    _check(d, {"X": xv}, {"Q": (n, c, ho, ho)}, exact=True)


def test_generated_rule_kernels_in_the_attention_graph(monkeypatch):
    b, s, dh = 2, 128, 64
    d = _attention_dag(b, s, dh, 0.125)
    rng = port.Rng(523)
    # the Z sums (128 per row) run as GROUP kernels: float association differs
    kinds = _generated_vs_interpreter(monkeypatch, d, {n: rng.tensor((b, s, dh)) for n in ("Q", "Kt", "V")},
                                      {"O": (b, s, dh)}, bitwise=False)
    assert kinds[1:5] == ["rule-generated"] * 4
