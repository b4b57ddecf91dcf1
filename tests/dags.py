"""DAG constructions for the BASELINE configs, written the way a user of the
reference API would: a reference builder (matmul_dag / conv2d_im2col_dag)
plus hand-appended epilogue nodes (validate() only needs loads
to reference earlier nodes, compute_ir.cpp:77-90)."""
from paper_2210_09603_b200 import (Axis, ComputeDAG, DType, TensorNode, add, conv2d_im2col_dag, gelu_tanh,
                                   load, matmul_dag, mul, relu, fimm, var)


def matmul_epilogue_dag(m, n, k, dtype=DType.F32, bias=True, act="relu"):
    """config 1: D[i,j] = act(C[i,j] + Bias[j])."""
    d = matmul_dag(m, n, k, dtype)
    v = load("C", [var("i"), var("j")])
    if bias:
        d.add_input("Bias", [n], dtype)
        v = add(v, load("Bias", [var("j")]))
    if act == "relu":
        v = relu(v)
    elif act == "gelu":
        v = gelu_tanh(v)
    d.add_compute("D", [Axis("i", m), Axis("j", n)], v, dtype)
    d.outputs = ["D"]
    return d


def batched_matmul_scale_dag(b, m, n, k, scale=0.125, dtype=DType.F32, kt_layout="bkn"):
    """config 2: P[b,i,j] = scale * sum_k Q[b,i,k] * K[b,.,.] with K given as
    KT[b,k,j] (kt_layout 'bkn', the reference matmul B[K,N] orientation) or
    Kmat[b,j,k] ('bnk', the natural attention layout)."""
    d = ComputeDAG()
    d.add_input("Q", [b, m, k], dtype)
    if kt_layout == "bkn":
        d.add_input("KT", [b, k, n], dtype)
        rhs = load("KT", [var("b"), var("k"), var("j")])
    else:
        d.add_input("Kmat", [b, n, k], dtype)
        rhs = load("Kmat", [var("b"), var("j"), var("k")])
    d.nodes.append(TensorNode("S", [b, m, n], dtype, "reduce", [Axis("b", b), Axis("i", m), Axis("j", n)],
                              [Axis("k", k)], value=mul(load("Q", [var("b"), var("i"), var("k")]), rhs)))
    d.add_compute("P", [Axis("b", b), Axis("i", m), Axis("j", n)],
                  mul(load("S", [var("b"), var("i"), var("j")]), fimm(scale)), dtype)
    d.outputs = ["P"]
    return d


def conv_bn_relu_dag(n, c, h, w, f, kh, kw, stride, pad, dtype=DType.F32):
    """config 3: Z = relu(Out[n,p,oh,ow] * Scale[p] + Shift[p]) on conv2d_im2col_dag."""
    d = conv2d_im2col_dag(n, c, h, w, f, kh, kw, stride, pad, dtype)
    out = d.at("Out")
    d.add_input("Scale", [f], dtype)
    d.add_input("Shift", [f], dtype)
    ax = [Axis(a.name, a.extent) for a in out.axes]
    x = load("Out", [var("n"), var("p"), var("oh"), var("ow")])
    d.add_compute("Z", ax, relu(add(mul(x, load("Scale", [var("p")])), load("Shift", [var("p")]))), dtype)
    d.outputs = ["Z"]
    return d


def ffn_dag(t, dm, dff, dtype=DType.F32):
    """config 4: H = gelu_tanh(X W1 + b1); O = H W2 + b2 + X."""
    d = ComputeDAG()
    d.add_input("X", [t, dm], dtype)
    d.add_input("W1", [dm, dff], dtype)
    d.add_input("b1", [dff], dtype)
    d.add_input("W2", [dff, dm], dtype)
    d.add_input("b2", [dm], dtype)
    d.nodes.append(TensorNode("H0", [t, dff], dtype, "reduce", [Axis("t", t), Axis("f", dff)], [Axis("k", dm)],
                              value=mul(load("X", [var("t"), var("k")]), load("W1", [var("k"), var("f")]))))
    d.add_compute("H", [Axis("t", t), Axis("f", dff)],
                  gelu_tanh(add(load("H0", [var("t"), var("f")]), load("b1", [var("f")]))), dtype)
    d.nodes.append(TensorNode("O0", [t, dm], dtype, "reduce", [Axis("t", t), Axis("d", dm)], [Axis("k", dff)],
                              value=mul(load("H", [var("t"), var("k")]), load("W2", [var("k"), var("d")]))))
    d.add_compute("O", [Axis("t", t), Axis("d", dm)],
                  add(add(load("O0", [var("t"), var("d")]), load("b2", [var("d")])), load("X", [var("t"), var("d")])),
                  dtype)
    d.outputs = ["O"]
    return d
