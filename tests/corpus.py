"""Shared test corpora: small instances of the BASELINE config DAGs, task
mappings and operator-classification cases (used by the golden generator and
the CPU parity tests)."""
import random

from oracle import port
from paper_2210_09603_b200 import (Axis, ComputeDAG, DType, TensorNode, add, div, fimm, imm, load, mod, mul,
                                   relu, select, sub, var, lt, ge, land, conv2d_im2col_dag, reshape_dag,
                                   transpose_dag, batchnorm_inference_dag, matmul_dag)

from dags import batched_matmul_scale_dag, conv_bn_relu_dag, ffn_dag, matmul_epilogue_dag


def dag_cases():
    """(name, dag, inputs, out_shapes) — small, seeded instances of every config chain."""
    cases = []
    r = port.Rng(1)
    m, n, k = 16, 12, 20
    for exact in (False, True):
        dt = DType.I32 if exact else DType.F32
        dag = matmul_epilogue_dag(m, n, k, dt)
        ins = {"A": r.tensor((m, k), exact), "B": r.tensor((k, n), exact), "Bias": r.tensor((n,), exact)}
        cases.append((f"matmul_bias_relu_{'i32' if exact else 'f32'}", dag, ins, {"D": (m, n)}))
    dag = matmul_epilogue_dag(8, 9, 10, act="gelu")
    ins = {"A": r.tensor((8, 10)), "B": r.tensor((10, 9)), "Bias": r.tensor((9,))}
    cases.append(("matmul_bias_gelu", dag, ins, {"D": (8, 9)}))
    dag = batched_matmul_scale_dag(2, 8, 8, 4)
    cases.append(("batched_scale", dag, {"Q": r.tensor((2, 8, 4)), "KT": r.tensor((2, 4, 8))}, {"P": (2, 8, 8)}))
    for g in [(1, 3, 7, 7, 4, 3, 3, 2, 1), (2, 2, 5, 6, 3, 1, 1, 1, 0), (1, 4, 6, 6, 2, 3, 3, 1, 1),
              (1, 3, 9, 9, 2, 7, 7, 2, 3)]:
        n_, c, h, w, f, kh, kw, s, p = g
        dag = conv_bn_relu_dag(n_, c, h, w, f, kh, kw, s, p)
        ho, wo = port.conv_out_extent(h, kh, s, p), port.conv_out_extent(w, kw, s, p)
        ins = {"X": r.tensor((n_, c, h, w)), "W": r.tensor((f, c, kh, kw)), "Scale": r.tensor((f,)),
               "Shift": r.tensor((f,))}
        cases.append((f"conv_bn_relu_{'_'.join(map(str, g))}", dag, ins, {"Z": (n_, f, ho, wo)}))
    dag = conv2d_im2col_dag(1, 2, 5, 5, 3, 3, 3, 2, 1)
    cases.append(("im2col_col", dag, {"X": r.tensor((1, 2, 5, 5)), "W": r.tensor((3, 2, 3, 3))},
                  {"Col": (18, 9), "Out": (1, 3, 3, 3)}))
    dag = ffn_dag(4, 8, 16)
    ins = {"X": r.tensor((4, 8)), "W1": r.tensor((8, 16)), "b1": r.tensor((16,)), "W2": r.tensor((16, 8)),
           "b2": r.tensor((8,))}
    cases.append(("ffn", dag, ins, {"O": (4, 8)}))
    return cases


def mapping_corpus():
    texts = ["repeat(2, 2)", "repeat(1)", "repeat(4, 1)", "spatial(2, 2)", "spatial(16, 8)",
             "repeat(4, 1) * spatial(16, 8)", "spatial(2) * repeat(2)", "repeat(2, 2) * spatial(2, 2)",
             "spatial(4, 2) * repeat(2, 2) * spatial(4, 8) * repeat(4, 4)",
             "spatial(2, 1) * repeat(1, 2)", "repeat(3, 1, 2) * spatial(2, 2, 1) * repeat(1, 3, 1)",
             "custom(workers=2, shape=(2, 2), table=[[(0, 0), (1, 1)], [(0, 1), (1, 0)]])",
             "custom(workers=2, shape=(4), table=[[(3), (0)], [(1), (2)]]) * spatial(2)",
             "(repeat(2) * spatial(3)) * (spatial(2) * repeat(2))"]
    rng = random.Random(7)
    for _ in range(40):
        dim = rng.randint(1, 3)
        atoms = []
        for _ in range(rng.randint(1, 4)):
            kind = rng.choice(["repeat", "spatial"])
            atoms.append(f"{kind}({', '.join(str(rng.randint(1, 4)) for _ in range(dim))})")
        texts.append(" * ".join(atoms))
    return texts


def _dag(nodes, inputs, outputs):
    return ComputeDAG(nodes, inputs, outputs).to_json()


def classify_corpus():
    """(name, dag_json, node) cases for fusion-legality parity with the reference."""
    out = []
    d = conv2d_im2col_dag(2, 3, 6, 6, 4, 3, 3, 1, 1)
    for nd in ("Col", "Wf", "Y", "Out"):
        out.append((f"conv:{nd}", d.to_json(), nd))
    d = matmul_dag(4, 5, 6)
    out.append(("matmul:C", d.to_json(), "C"))
    for a, b in [([100], [2, 50]), ([2, 50], [100]), ([4, 12, 8], [4, 96]), ([4, 96], [4, 12, 8]), ([6], [6])]:
        out.append((f"reshape:{a}->{b}", reshape_dag(a, b).to_json(), "Y"))
    out.append(("transpose:0213", transpose_dag([2, 3, 4, 5], [0, 2, 1, 3]).to_json(), "Y"))
    out.append(("transpose:10", transpose_dag([3, 1], [1, 0]).to_json(), "Y"))
    out.append(("batchnorm", batchnorm_inference_dag(2, 3, 4, 4).to_json(), "Y"))
    for name, dag in [("cfg1", matmul_epilogue_dag(4, 5, 6)), ("cfg2", batched_matmul_scale_dag(2, 4, 4, 3)),
                      ("cfg3", conv_bn_relu_dag(1, 2, 5, 5, 3, 3, 3, 1, 1)), ("cfg4", ffn_dag(3, 4, 6))]:
        for n in dag.nodes:
            if n.kind != "input":
                out.append((f"{name}:{n.name}", dag.to_json(), n.name))
    # hand-written cases
    X = TensorNode("X", [100])
    out.append(("reverse", _dag([X, TensorNode("Y", [100], kind="compute", axes=[Axis("i", 100)],
                                               value=mul(load("X", [sub(imm(99), var("i"))]), fimm(2.0)))],
                                ["X"], ["Y"]), "Y"))
    X2 = TensorNode("X", [4])
    out.append(("broadcast", _dag([X2, TensorNode("Y", [4, 3], kind="compute", axes=[Axis("i", 4), Axis("j", 3)],
                                                  value=load("X", [var("i")]))], ["X"], ["Y"]), "Y"))
    X3 = TensorNode("X", [4, 4])
    out.append(("two_accesses", _dag([X3, TensorNode("Y", [4, 4], kind="compute", axes=[Axis("i", 4), Axis("j", 4)],
                                                     value=add(load("X", [var("i"), var("j")]),
                                                               load("X", [var("j"), var("i")])))], ["X"], ["Y"]), "Y"))
    out.append(("same_access_twice", _dag([X3, TensorNode("Y", [4, 4], kind="compute", axes=[Axis("i", 4), Axis("j", 4)],
                                                          value=mul(load("X", [var("i"), var("j")]),
                                                                    load("X", [var("i"), var("j")])))],
                                          ["X"], ["Y"]), "Y"))
    X4 = TensorNode("X", [8])
    out.append(("guarded", _dag([X4, TensorNode("Y", [10], kind="compute", axes=[Axis("i", 10)],
                                                value=select(land(ge(sub(var("i"), imm(1)), imm(0)),
                                                                  lt(sub(var("i"), imm(1)), imm(8))),
                                                             load("X", [sub(var("i"), imm(1))]), fimm(0.0)))],
                                ["X"], ["Y"]), "Y"))
    out.append(("divmod", _dag([X4, TensorNode("Y", [2, 4], kind="compute", axes=[Axis("i", 2), Axis("j", 4)],
                                               value=load("X", [add(mul(var("i"), imm(4)), var("j"))]))],
                               ["X"], ["Y"]), "Y"))
    out.append(("stride2", _dag([X4, TensorNode("Y", [4], kind="compute", axes=[Axis("i", 4)],
                                                value=load("X", [mul(var("i"), imm(2))]))], ["X"], ["Y"]), "Y"))
    X5 = TensorNode("X", [1, 6])
    out.append(("unit_axis", _dag([X5, TensorNode("Y", [1, 6], kind="compute", axes=[Axis("a", 1), Axis("b", 6)],
                                                  value=load("X", [mul(var("a"), imm(3)), var("b")]))],
                                  ["X"], ["Y"]), "Y"))
    out.append(("mod_index", _dag([X4, TensorNode("Y", [8], kind="compute", axes=[Axis("i", 8)],
                                                  value=load("X", [mod(add(var("i"), imm(3)), imm(8))]))],
                                  ["X"], ["Y"]), "Y"))
    out.append(("div_index", _dag([X4, TensorNode("Y", [4], kind="compute", axes=[Axis("i", 4)],
                                                  value=load("X", [div(var("i"), imm(1))]))], ["X"], ["Y"]), "Y"))
    return out
