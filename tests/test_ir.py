"""Host-side IR parity with the reference (CPU only): builders, classify
(fusion legality), DAG validation, partition and the fused-kernel plans."""
import json
import os

import pytest

import oracle
from paper_2210_09603_b200 import (Axis, ComputeDAG, DType, OpClass, Plan, ScheduleConfig, TaskmapError, TensorNode,
                                   classify, load, matmul_dag, partition, var, workloads)
from paper_2210_09603_b200 import taskmap as T

from dags import batched_matmul_scale_dag, conv_bn_relu_dag, ffn_dag, matmul_epilogue_dag

HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))


@pytest.mark.parametrize("key", sorted(META["builders"]))
def test_builders_match_reference(key):
    """Same DAG structure and expression trees as compute_ir.cpp:496-733."""
    kind, args = key.split(":")
    args = [int(a) for a in args.split(",")]
    mine = json.loads(T._build(kind, args).to_json())
    ref = json.loads(META["builders"][key])
    assert mine == ref


@pytest.mark.parametrize("case", META["classify"], ids=[c["name"] for c in META["classify"]])
def test_classify_matches_reference(case):
    """classify (compute_ir.cpp:222-243) decides fusion legality: must agree exactly."""
    dag = ComputeDAG.from_json(case["dag"])
    assert int(classify(dag, case["node"])) == case["class"]


def test_classify_probe_decisions():
    """matmul C reduction; conv Col/Wf injective; Out bijective; reshape split
    bijective but merge injective; transpose and BN bijective."""
    conv = T.conv2d_im2col_dag(2, 3, 6, 6, 4, 3, 3, 1, 1)
    assert [classify(conv, n) for n in ("Col", "Wf", "Y", "Out")] == [
        OpClass.Injective, OpClass.Injective, OpClass.Reduction, OpClass.Bijective]
    assert classify(T.reshape_dag([100], [2, 50]), "Y") == OpClass.Bijective
    assert classify(T.reshape_dag([2, 50], [100]), "Y") == OpClass.Injective
    assert classify(T.transpose_dag([2, 3, 4, 5], [0, 2, 1, 3]), "Y") == OpClass.Bijective


def test_validate_errors_match_reference():
    bad = [
        ComputeDAG([TensorNode("X", [4]), TensorNode("X", [4], kind="compute", axes=[Axis("i", 4)],
                                                     value=load("X", [var("i")]))], ["X"], ["X"]),
        ComputeDAG([TensorNode("Y", [4], kind="compute", axes=[Axis("i", 4)], value=load("Z", [var("i")]))], [], ["Y"]),
        ComputeDAG([TensorNode("X", [4]), TensorNode("Y", [4], kind="compute", axes=[Axis("i", 4)],
                                                     value=load("X", [var("j")]))], ["X"], ["Y"]),
        ComputeDAG([TensorNode("X", [4]), TensorNode("Y", [4], kind="compute", axes=[Axis("i", 3)],
                                                     value=load("X", [var("i")]))], ["X"], ["Y"]),
    ]
    for d in bad:
        with pytest.raises(TaskmapError) as mine:
            classify(d, d.nodes[-1].name)
        if oracle.ref_available():
            with pytest.raises(oracle.RefError) as ref:
                oracle.ref_validate(d.to_json())
            assert str(mine.value) == str(ref.value)


def test_partition_config_chains():
    """Conv->BN->ReLU is one subgraph (im2col + filter prologues,
    reshape + BN/ReLU epilogue); the FFN chain is two anchors."""
    p = partition(conv_bn_relu_dag(1, 3, 8, 8, 4, 3, 3, 1, 1))
    assert p == [{"anchor": "Y", "prologue": ["Wf", "Col"], "epilogue": ["Out", "Z"], "output": "Z"}]
    p = partition(ffn_dag(8, 16, 32))
    assert [s["anchor"] for s in p] == ["H0", "O0"] and p[0]["epilogue"] == ["H"] and p[1]["epilogue"] == ["O"]
    p = partition(matmul_epilogue_dag(4, 4, 4))
    assert p == [{"anchor": "C", "prologue": [], "epilogue": ["D"], "output": "D"}]


def test_plans_lower_config_chains():
    """Fused-kernel plans (no GPU needed to plan): loaders, epilogue programs, remaps."""
    d = Plan(conv_bn_relu_dag(2, 64, 8, 8, 64, 3, 3, 1, 1)).describe()["kernels"][0]
    assert d["A"] == "im2col(X)" and d["B"] == "filter(W)"
    assert [o["kind"] for o in d["ops"]] == [19, 16, 32]      # MUL_T Scale, ADD_T Shift, RELU
    d = Plan(batched_matmul_scale_dag(6, 128, 128, 64)).describe()["kernels"][0]
    assert d["batch"] == 6 and [o["kind"] for o in d["ops"]] == [4]  # MUL_C 0.125
    d = Plan(ffn_dag(64, 32, 128)).describe()
    assert len(d["kernels"]) == 2 and d["intermediates"] == ["H"]
    assert [o["kind"] for o in d["kernels"][0]["ops"]] == [16, 33]   # bias, GELU (tanh form matched)
    assert [o["kind"] for o in d["kernels"][1]["ops"]] == [16, 16]   # bias, residual


def test_fig11_prologue_epilogue_remap():
    """PAPER Fig. 11 / SPEC.md:376,385: "the access of A[99 - i] will be replaced by
    C[99 - i] * 2.0" -- an arithmetic prologue over a reversed re-index, lowered to the
    operand's address map plus a prologue op list (MUL_C 2.0) for the gather loader --
    and the epilogue stores y*3 at (i/50, i%50)."""
    from paper_2210_09603_b200 import fimm, mul, sub, imm
    d = ComputeDAG()
    d.add_input("C", [100, 8])
    d.add_input("B", [8, 4])
    d.nodes.append(TensorNode("A", [100, 8], kind="compute", axes=[Axis("i", 100), Axis("k", 8)],
                              value=mul(load("C", [sub(imm(99), var("i")), var("k")]), fimm(2.0))))
    d.nodes.append(TensorNode("Y", [100, 4], kind="reduce", axes=[Axis("i", 100), Axis("j", 4)],
                              reduce_axes=[Axis("k", 8)], value=mul(load("A", [var("i"), var("k")]),
                                                                     load("B", [var("k"), var("j")]))))
    d.nodes.append(TensorNode("D", [2, 50, 4], kind="compute", axes=[Axis("a", 2), Axis("b", 50), Axis("j", 4)],
                              value=mul(load("Y", [T.add(mul(var("a"), imm(50)), var("b")), var("j")]), fimm(3.0))))
    d.outputs = ["D"]
    assert partition(d) == [{"anchor": "Y", "prologue": ["A"], "epilogue": ["D"], "output": "D"}]
    k = Plan(d).describe()["kernels"][0]
    assert k["A"].startswith("C[99 - __row") and k["A"].endswith("|> op4(2.000000)")  # MUL_C 2.0
    assert [o["kind"] for o in k["ops"]] == [4] and k["ops"][0]["c"] == 3  # epilogue MUL_C 3.0


def test_relu_prologue_and_rejected_prologues():
    """SPEC.md:368 ReLU -> matmul -> matmul: the ReLU is the first anchor's prologue op.
    Prologues the gather loader cannot apply (two input elements, a tensor side
    operand) are refused with TM_ERR_UNSUPPORTED."""
    from paper_2210_09603_b200 import relu, add
    def dag(value):
        d = ComputeDAG()
        d.add_input("X", [16, 8])
        d.add_input("W", [8, 4])
        d.add_input("V", [16, 8])
        d.nodes.append(TensorNode("R", [16, 8], kind="compute", axes=[Axis("i", 16), Axis("k", 8)], value=value))
        d.nodes.append(TensorNode("Y", [16, 4], kind="reduce", axes=[Axis("i", 16), Axis("j", 4)],
                                  reduce_axes=[Axis("k", 8)], value=T.mul(load("R", [var("i"), var("k")]),
                                                                           load("W", [var("k"), var("j")]))))
        d.outputs = ["Y"]
        return d
    x = load("X", [var("i"), var("k")])
    k = Plan(dag(relu(x))).describe()["kernels"][0]
    assert k["prologue"] == ["R"] and k["A"].endswith("|> op32(0.000000)")  # RELU
    # a prologue the loader cannot apply (two input elements) is materialised by a
    # rule-based kernel first; the GEMM then reads it
    ks = Plan(dag(add(x, load("V", [var("i"), var("k")])))).describe()["kernels"]
    assert [k["kind"] for k in ks] == ["rule", "gemm"]
    assert ks[0]["root"] == "R" and ks[1]["prologue"] == [] and ks[1]["A"].startswith("R[")


def test_schedule_space_size_and_agnostic():
    """50 <= |space| <= 200, identical for every shape."""
    from paper_2210_09603_b200 import schedule_space
    s = schedule_space("matmul")
    assert 50 <= len(s) <= 200
    conv = schedule_space("conv2d")  # + the halo kernel family
    assert conv[:len(s)] == s and len(conv) == len(s) + 1 and conv[-1].math == "halo"
    assert len({(c.block_m, c.block_n, c.split_k, c.pipeline, c.raster, c.grid) for c in s}) == len(s)


def test_reduce_schedule_space():
    """schedule_space(op_kind) for op_kind in {matmul, reduce}."""
    from paper_2210_09603_b200 import schedule_space
    s = schedule_space("reduce")
    assert [c.threads_per_block for c in s] == [128, 256, 512, 64, 32]


def test_non_matmul_reduction_plans_the_reduce_template():
    """a max reduction is not a matrix product -> reduce_template."""
    d = ComputeDAG()
    d.add_input("X", [4, 4])
    d.nodes.append(TensorNode("Y", [4], kind="reduce", axes=[Axis("i", 4)], reduce_axes=[Axis("j", 4)],
                              combiner=T.Combiner.Max, value=load("X", [var("i"), var("j")])))
    d.outputs = ["Y"]
    (k,) = Plan(d).describe()["kernels"]
    assert k["kind"] == "reduce" and k["root"] == "Y" and k["reduce"] == 4


def test_anchor_free_chain_fuses_into_one_rule_kernel():
    """the elementwise chain a*2+1 (then ReLU) is one rule-based kernel."""
    from paper_2210_09603_b200 import relu, add, mul, fimm
    d = ComputeDAG()
    d.add_input("A", [1000])
    d.add_compute("T1", [Axis("i", 1000)], mul(load("A", [var("i")]), fimm(2.0)))
    d.add_compute("T2", [Axis("i", 1000)], add(load("T1", [var("i")]), fimm(1.0)))
    d.add_compute("T3", [Axis("i", 1000)], relu(load("T2", [var("i")])))
    d.outputs = ["T3"]
    sgs = T.partition(d)
    assert len(sgs) == 1 and sgs[0]["output"] == "T3" and sgs[0]["prologue"] == ["T1", "T2"]
    (k,) = Plan(d).describe()["kernels"]
    assert k["kind"] == "rule" and k["inlined"] == ["T1", "T2"] and "T1" not in k["expr"]


def test_workload_flops():
    assert abs(sum(L.flops(32) * L.count for L in workloads.RESNET50) / 1e9 - 261.6) < 0.1
