"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference arithmetic.

Each function restates the reference's definition for one BASELINE config in
float64 (the reference evaluates f32 DAGs in double, tensor.hpp:12-18) and
cites the reference lines it follows.  Pinned against oracle/_ref (the real
reference_eval) and the golden fixtures by tests/test_oracle.py.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


class Rng:
    """splitmix64 stream of taskmap::Rng (proj/src/tensor.cpp:42-59), vectorised."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed if seed else 0x9E3779B97F4A7C15)

    def next(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(1, n + 1, dtype=np.uint64)
            z = self.state + k * GOLDEN
            self.state = self.state + np.uint64(n) * GOLDEN
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            return z ^ (z >> np.uint64(31))

    def uniform_real(self, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        u = (self.next(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53   # tensor.cpp:56-59
        return lo + u * (hi - lo)

    def uniform_int(self, n: int, lo: int = -8, hi: int = 8) -> np.ndarray:
        span = np.uint64(hi - lo + 1)                                          # tensor.cpp:51-54
        return (lo + (self.next(n) % span).astype(np.int64)).astype(np.float64)

    def tensor(self, shape, is_int: bool = False) -> np.ndarray:
        """random_tensor (tensor.cpp:61-69): f32 -> U(-1,1), i32 -> U{-8..8}."""
        n = int(np.prod(shape))
        v = self.uniform_int(n) if is_int else self.uniform_real(n)
        return v.reshape(shape)


def max_rel_error(a, b) -> float:
    """max |a-b| / max(1, |b|) (tensor.cpp:71-86)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def fold_batchnorm_params(gamma, beta, mean, var, eps):
    """compute_ir.cpp:721-733: scale = gamma/sqrt(var+eps), shift = beta - mean*scale."""
    s = np.asarray(gamma, np.float64) / np.sqrt(np.asarray(var, np.float64) + eps)
    return s, np.asarray(beta, np.float64) - np.asarray(mean, np.float64) * s


def matmul(a, b):
    """matmul_dag (compute_ir.cpp:496-515): C[i,j] = sum_k A[i,k] B[k,j]."""
    return np.asarray(a, np.float64) @ np.asarray(b, np.float64)


def matmul_bias_relu(a, b, bias):
    """config 1: D[i,j] = relu(C[i,j] + Bias[j])."""
    return np.maximum(matmul(a, b) + np.asarray(bias, np.float64)[None, :], 0.0)


def batched_matmul_scale(q, kt, scale):
    """config 2: S[b,i,j] = scale * sum_k Q[b,i,k] KT[b,k,j] (GridReduce with a batch axis)."""
    return scale * np.einsum("bik,bkj->bij", np.asarray(q, np.float64), np.asarray(kt, np.float64))


def conv_out_extent(i, k, s, p):
    """compute_ir.hpp:117-119."""
    return (i + 2 * p - k) // s + 1


def im2col(x, kh, kw, stride, pad):
    """Col[r, s] of conv2d_im2col_dag (compute_ir.cpp:532-557), reference index order:
    r -> (c = r/(kh kw), fh = (r/kw)%kh, fw = r%kw), s -> (n = s/(ho wo), oh = (s/wo)%ho, ow = s%wo),
    zero outside the padded image."""
    x = np.asarray(x, np.float64)
    n, c, h, w = x.shape
    ho, wo = conv_out_extent(h, kh, stride, pad), conv_out_extent(w, kw, stride, pad)
    r = np.arange(c * kh * kw)
    s = np.arange(n * ho * wo)
    ch, fh, fw = r // (kh * kw), (r // kw) % kh, r % kw
    img, oh, ow = s // (ho * wo), (s // wo) % ho, s % wo
    ih = (oh * stride - pad)[None, :] + fh[:, None]
    iw = (ow * stride - pad)[None, :] + fw[:, None]
    ok = (ih >= 0) & (ih < h) & (iw >= 0) & (iw < w)
    col = x[img[None, :], ch[:, None], np.clip(ih, 0, h - 1), np.clip(iw, 0, w - 1)]
    return np.where(ok, col, 0.0)


def conv2d_nchw(x, wt, stride, pad):
    """conv2d_im2col_dag output Out[n,p,oh,ow] = Y[p, (n*ho+oh)*wo+ow], Y = Wf @ Col (compute_ir.cpp:558-592)."""
    x = np.asarray(x, np.float64)
    wt = np.asarray(wt, np.float64)
    n, c, h, w = x.shape
    f, _, kh, kw = wt.shape
    ho, wo = conv_out_extent(h, kh, stride, pad), conv_out_extent(w, kw, stride, pad)
    y = wt.reshape(f, c * kh * kw) @ im2col(x, kh, kw, stride, pad)
    return y.reshape(f, n, ho, wo).transpose(1, 0, 2, 3)


def conv_bn_relu(x, wt, scale, shift, stride, pad):
    """config 3: Z[n,p,oh,ow] = relu(Out[n,p,oh,ow] * Scale[p] + Shift[p]) (batchnorm_inference_dag, :701-719)."""
    out = conv2d_nchw(x, wt, stride, pad)
    sc = np.asarray(scale, np.float64)[None, :, None, None]
    sh = np.asarray(shift, np.float64)[None, :, None, None]
    return np.maximum(out * sc + sh, 0.0)


def gelu_tanh(x):
    """The Exp/Div form of tanh-GELU used in the DAGs (the IR has no tanh, expr.hpp:16)."""
    x = np.asarray(x, np.float64)
    inner = 0.7978845608028654 * (x + 0.044715 * (x * x * x))
    with np.errstate(over="ignore"):
        t = 1.0 - 2.0 / (np.exp(2.0 * inner) + 1.0)
    return 0.5 * x * (1.0 + t)


def ffn(x, w1, b1, w2, b2, round_h=None):
    """config 4: H = gelu_tanh(X W1 + b1); O = H W2 + b2 + X.  round_h optionally models the
    device's bf16 storage of the intermediate H (the reference keeps it in double)."""
    h = gelu_tanh(matmul(x, w1) + np.asarray(b1, np.float64)[None, :])
    if round_h is not None:
        h = round_h(h)
    return matmul(h, w2) + np.asarray(b2, np.float64)[None, :] + np.asarray(x, np.float64)


def round_bf16(a) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (host-side rounding of inputs)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def round_tf32(a) -> np.ndarray:
    """Round-to-nearest-even to tf32 (10-bit mantissa), returned as float64."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(13)) & np.uint64(1)
    r = ((u + np.uint64(0xFFF) + lsb) >> np.uint64(13)) << np.uint64(13)
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
