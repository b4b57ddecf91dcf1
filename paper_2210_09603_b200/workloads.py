"""The BASELINE.json workloads as DAGs.

Every DAG is built like a user of the reference API would: a reference-style
builder (matmul_dag / conv2d_im2col_dag, compute_ir.cpp:496-597) plus
appended epilogue nodes.
"""
from dataclasses import dataclass
from typing import List

from .taskmap import (Axis, ComputeDAG, DType, TensorNode, add, conv2d_im2col_dag, fimm, gelu_tanh, load,
                      matmul_dag, mul, relu, var)


@dataclass(frozen=True)
class ConvLayer:
    name: str
    c: int
    h: int
    f: int
    k: int
    s: int
    p: int
    count: int

    def out_hw(self) -> int:
        return (self.h + 2 * self.p - self.k) // self.s + 1

    def gemm(self, batch: int):
        ho = self.out_hw()
        return batch * ho * ho, self.f, self.c * self.k * self.k  # M (pixels), N (filters), K

    def flops(self, batch: int) -> float:
        m, n, k = self.gemm(batch)
        return 2.0 * m * n * k


# torchvision ResNet-50 v1.5 conv layers: 24 shapes, 53 layers
RESNET50: List[ConvLayer] = [
    ConvLayer("conv1", 3, 224, 64, 7, 2, 3, 1),
    ConvLayer("l1.c1a", 64, 56, 64, 1, 1, 0, 1),
    ConvLayer("l1.c1", 256, 56, 64, 1, 1, 0, 2),
    ConvLayer("l1.c2", 64, 56, 64, 3, 1, 1, 3),
    ConvLayer("l1.c3", 64, 56, 256, 1, 1, 0, 3),
    ConvLayer("l1.ds", 64, 56, 256, 1, 1, 0, 1),
    ConvLayer("l2.c1a", 256, 56, 128, 1, 1, 0, 1),
    ConvLayer("l2.c2s", 128, 56, 128, 3, 2, 1, 1),
    ConvLayer("l2.c1", 512, 28, 128, 1, 1, 0, 3),
    ConvLayer("l2.c2", 128, 28, 128, 3, 1, 1, 3),
    ConvLayer("l2.c3", 128, 28, 512, 1, 1, 0, 4),
    ConvLayer("l2.ds", 256, 56, 512, 1, 2, 0, 1),
    ConvLayer("l3.c1a", 512, 28, 256, 1, 1, 0, 1),
    ConvLayer("l3.c2s", 256, 28, 256, 3, 2, 1, 1),
    ConvLayer("l3.c1", 1024, 14, 256, 1, 1, 0, 5),
    ConvLayer("l3.c2", 256, 14, 256, 3, 1, 1, 5),
    ConvLayer("l3.c3", 256, 14, 1024, 1, 1, 0, 6),
    ConvLayer("l3.ds", 512, 28, 1024, 1, 2, 0, 1),
    ConvLayer("l4.c1a", 1024, 14, 512, 1, 1, 0, 1),
    ConvLayer("l4.c2s", 512, 14, 512, 3, 2, 1, 1),
    ConvLayer("l4.c1", 2048, 7, 512, 1, 1, 0, 2),
    ConvLayer("l4.c2", 512, 7, 512, 3, 1, 1, 2),
    ConvLayer("l4.c3", 512, 7, 2048, 1, 1, 0, 3),
    ConvLayer("l4.ds", 1024, 14, 2048, 1, 2, 0, 1),
]

RESNET_BATCH = 32
BERT_TOKENS = 64 * 128     # batch 64 x seq 128
BERT_HIDDEN, BERT_FFN = 768, 3072
BERT_HEADS, BERT_SEQ, BERT_HEAD_DIM = 12 * 16, 128, 64


def conv_bn_relu_dag(layer: ConvLayer, batch: int, f: int = None, dtype: DType = DType.F32) -> ComputeDAG:
    """config 3: Z = relu(conv(X, W) * Scale[p] + Shift[p]) via conv2d_im2col_dag."""
    f = f or layer.f
    d = conv2d_im2col_dag(batch, layer.c, layer.h, layer.h, f, layer.k, layer.k, layer.s, layer.p, dtype)
    out = d.at("Out")
    d.add_input("Scale", [f], dtype)
    d.add_input("Shift", [f], dtype)
    x = load("Out", [var("n"), var("p"), var("oh"), var("ow")])
    d.add_compute("Z", [Axis(a.name, a.extent) for a in out.axes],
                  relu(add(mul(x, load("Scale", [var("p")])), load("Shift", [var("p")]))), dtype)
    d.outputs = ["Z"]
    return d


def ffn_dag(t: int, dm: int = BERT_HIDDEN, dff: int = BERT_FFN, dtype: DType = DType.F32) -> ComputeDAG:
    """config 4: H = gelu_tanh(X W1 + b1); O = H W2 + b2 + X."""
    d = ComputeDAG()
    for name, shape in (("X", [t, dm]), ("W1", [dm, dff]), ("b1", [dff]), ("W2", [dff, dm]), ("b2", [dm])):
        d.add_input(name, shape, dtype)
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


def attention_scores_dag(b: int, s: int = BERT_SEQ, dh: int = BERT_HEAD_DIM, scale: float = 0.125,
                         dtype: DType = DType.F32) -> ComputeDAG:
    """config 2a: S[b,i,j] = scale * sum_k Q[b,i,k] K[b,j,k] (softmax-free scale epilogue)."""
    d = ComputeDAG()
    d.add_input("Q", [b, s, dh], dtype)
    d.add_input("K", [b, s, dh], dtype)
    d.nodes.append(TensorNode("S0", [b, s, s], dtype, "reduce", [Axis("b", b), Axis("i", s), Axis("j", s)],
                              [Axis("k", dh)], value=mul(load("Q", [var("b"), var("i"), var("k")]),
                                                         load("K", [var("b"), var("j"), var("k")]))))
    d.add_compute("S", [Axis("b", b), Axis("i", s), Axis("j", s)], mul(load("S0", [var("b"), var("i"), var("j")]),
                                                                     fimm(scale)), dtype)
    d.outputs = ["S"]
    return d


def attention_context_dag(b: int, s: int = BERT_SEQ, dh: int = BERT_HEAD_DIM, dtype: DType = DType.F32) -> ComputeDAG:
    """config 2b: O[b,i,d] = sum_j P[b,i,j] V[b,j,d]."""
    d = ComputeDAG()
    d.add_input("P", [b, s, s], dtype)
    d.add_input("V", [b, s, dh], dtype)
    d.nodes.append(TensorNode("O", [b, s, dh], dtype, "reduce", [Axis("b", b), Axis("i", s), Axis("d", dh)],
                              [Axis("j", s)], value=mul(load("P", [var("b"), var("i"), var("j")]),
                                                        load("V", [var("b"), var("j"), var("d")]))))
    d.outputs = ["O"]
    return d


def matmul_bias_relu_dag(m: int, n: int, k: int, dtype: DType = DType.F32) -> ComputeDAG:
    """config 1: D = relu(A B + Bias)."""
    d = matmul_dag(m, n, k, dtype)
    d.add_input("Bias", [n], dtype)
    d.add_compute("D", [Axis("i", m), Axis("j", n)], relu(add(load("C", [var("i"), var("j")]),
                                                               load("Bias", [var("j")]))), dtype)
    d.outputs = ["D"]
    return d
