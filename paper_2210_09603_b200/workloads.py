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


# ---------------------------------------------------------------- network chain --
# ResNet-50 v1.5 as one chain of the tensor programs above:
# stem conv + max pool, 16 bottleneck blocks (1x1 -> 3x3 (stride) -> 1x1 with the
# residual add fused into the last conv's epilogue, downsample conv on the first
# block of each stage), global average pool, classifier GEMM.

def conv_bn_dag(layer: ConvLayer, batch: int, relu_out: bool = True, residual: bool = False,
                dtype: DType = DType.F32) -> ComputeDAG:
    """Z = [relu](conv(X, W) * Scale[p] + Shift[p] [+ R[n,p,oh,ow]]) -- the bottleneck's
    conv kinds: c1/c2 (ReLU), c3 (residual, then ReLU), downsample (neither)."""
    d = conv2d_im2col_dag(batch, layer.c, layer.h, layer.h, layer.f, layer.k, layer.k, layer.s, layer.p, dtype)
    out = d.at("Out")
    d.add_input("Scale", [layer.f], dtype)
    d.add_input("Shift", [layer.f], dtype)
    idx = [var("n"), var("p"), var("oh"), var("ow")]
    v = add(mul(load("Out", idx), load("Scale", [var("p")])), load("Shift", [var("p")]))
    if residual:
        ho = layer.out_hw()
        d.add_input("R", [batch, layer.f, ho, ho], dtype)
        v = add(v, load("R", idx))
    d.add_compute("Z", [Axis(a.name, a.extent) for a in out.axes], relu(v) if relu_out else v, dtype)
    d.outputs = ["Z"]
    return d


def maxpool_dag(batch: int, c: int, h: int, k: int = 3, s: int = 2, p: int = 1,
                dtype: DType = DType.F32) -> ComputeDAG:
    """Y[n,c,y,x] = max over the k x k window at (y*s - p, x*s - p); out-of-image taps
    are excluded by a guard (reduce_template with the Max combiner)."""
    from .taskmap import Combiner, ge, land, lt, select, sub
    from .taskmap import imm as iimm
    ho = (h + 2 * p - k) // s + 1
    d = ComputeDAG()
    d.add_input("X", [batch, c, h, h], dtype)
    nn, cc, y, x, r, q = var("n"), var("c"), var("y"), var("x"), var("r"), var("q")
    iy = sub(add(mul(y, iimm(s)), r), iimm(p))
    ix = sub(add(mul(x, iimm(s)), q), iimm(p))
    inb = land(land(ge(iy, iimm(0)), lt(iy, iimm(h))), land(ge(ix, iimm(0)), lt(ix, iimm(h))))
    d.nodes.append(TensorNode("Y", [batch, c, ho, ho], dtype, "reduce",
                              [Axis("n", batch), Axis("c", c), Axis("y", ho), Axis("x", ho)],
                              [Axis("r", k), Axis("q", k)], combiner=Combiner.Max,
                              value=select(inb, load("X", [nn, cc, iy, ix]), fimm(-3.0e38))))
    d.outputs = ["Y"]
    return d


def avgpool_dag(batch: int, c: int, h: int, dtype: DType = DType.F32) -> ComputeDAG:
    """G[n,c] = mean over the h x h map (a sum reduction of X / h^2)."""
    d = ComputeDAG()
    d.add_input("X", [batch, c, h, h], dtype)
    d.nodes.append(TensorNode("G", [batch, c], dtype, "reduce", [Axis("n", batch), Axis("c", c)],
                              [Axis("y", h), Axis("x", h)],
                              value=mul(load("X", [var("n"), var("c"), var("y"), var("x")]), fimm(1.0 / (h * h)))))
    d.outputs = ["G"]
    return d


def linear_dag(m: int, n: int, k: int, dtype: DType = DType.F32) -> ComputeDAG:
    """Y = A B + Bias (the classifier)."""
    d = matmul_dag(m, n, k, dtype)
    d.add_input("Bias", [n], dtype)
    d.add_compute("D", [Axis("i", m), Axis("j", n)], add(load("C", [var("i"), var("j")]), load("Bias", [var("j")])),
                  dtype)
    d.outputs = ["D"]
    return d


@dataclass(frozen=True)
class ChainStage:
    """One kernel group of the network chain: `kind` in conv / maxpool / avgpool /
    linear; `src` / `res` name the activations it reads, `dst` the one it writes;
    `layer` is the RESNET50 table entry whose tuned schedule a conv reuses."""
    kind: str
    dst: str
    src: str
    res: str = ""
    conv: ConvLayer = None
    layer: str = ""
    relu: bool = True


def resnet50_stages(image: int = 224, classes: int = 1000, blocks=(3, 4, 6, 3)) -> List[ChainStage]:
    """The chain's stages in execution order.  At image 224 every conv equals the
    RESNET50 table entry named in `layer` (same shape; its tuned schedule applies)."""
    st = []
    h = image
    stem = ConvLayer("conv1", 3, h, 64, 7, 2, 3, 1)
    st.append(ChainStage("conv", "stem", "input", conv=stem, layer="conv1"))
    h = stem.out_hw()
    st.append(ChainStage("maxpool", "pool", "stem"))
    h = (h + 2 - 3) // 2 + 1
    cin, cur = 64, "pool"
    for li, (nb, width) in enumerate(zip(blocks, (64, 128, 256, 512))):
        for b in range(nb):
            first = b == 0
            s = 2 if first and li > 0 else 1
            pre = f"l{li + 1}.b{b}"
            c1 = ConvLayer(f"{pre}.c1", cin, h, width, 1, 1, 0, 1)
            c1_tab = "l1.c1a" if (li == 0 and first) else (f"l{li + 1}.c1a" if first else f"l{li + 1}.c1")
            st.append(ChainStage("conv", f"{pre}.c1", cur, conv=c1, layer=c1_tab))
            c2 = ConvLayer(f"{pre}.c2", width, h, width, 3, s, 1, 1)
            st.append(ChainStage("conv", f"{pre}.c2", f"{pre}.c1", conv=c2,
                                 layer=f"l{li + 1}.c2s" if s == 2 else f"l{li + 1}.c2"))
            ho = c2.out_hw()
            res = cur
            if first:
                ds = ConvLayer(f"{pre}.ds", cin, h, width * 4, 1, s, 0, 1)
                st.append(ChainStage("conv", f"{pre}.ds", cur, conv=ds, layer=f"l{li + 1}.ds", relu=False))
                res = f"{pre}.ds"
            c3 = ConvLayer(f"{pre}.c3", width, ho, width * 4, 1, 1, 0, 1)
            st.append(ChainStage("conv", f"{pre}.c3", f"{pre}.c2", res=res, conv=c3, layer=f"l{li + 1}.c3"))
            cur, cin, h = f"{pre}.c3", width * 4, ho
    st.append(ChainStage("avgpool", "gap", cur))
    st.append(ChainStage("linear", "logits", "gap"))
    return st
