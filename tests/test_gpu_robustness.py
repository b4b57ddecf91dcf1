"""Round-2 regressions on the GPU:

* the round-1 intermittent hang (loader warps polling ring slots they did not
  own, no producer tail) on its fastest repro, the CTA-pair BN=128 residual GEMM,
  plus the split-K schedules that used to be pruned;
* operand / output views whose batch stride is smaller than one batch's rows
  (heads interleaved inside a row) -- they must not be described as TMA tiles;
* fp16 operands: kind::f16 with the fp16 a/b format (round 1 fed fp16 bits to an
  MMA told they were bf16), K-major and MN-major B, CTA pairs, split-K, conv.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import port
from paper_2210_09603_b200 import DType, Plan, ScheduleConfig, TaskmapError

from dags import batched_matmul_scale_dag, conv_bn_relu_dag, matmul_epilogue_dag
from gpu_util import dev, run

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_round1_hang_repro_runs_clean():
    """pair BN=128 on the FFN's residual GEMM hung within ~20 x 5 launches on the
    round-1 build (gpurun_out/r02p1); it must now finish 60 x 5 under a watchdog."""
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "hang_probe.py"), "--case", "res", "--tokens", "4096",
           "--cfgs", "pair128,pair128sk2,bn64sk2,sk4", "--reps", "60", "--watchdog", "10"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "all configs completed" in r.stdout, r.stdout + r.stderr


def _torch():
    import torch
    return torch


def test_heads_interleaved_batch_views_exact():
    """Q, K stored [S, H, D] (one token's heads side by side), bound as logical [H, S, D]
    with strides (D, H*D, 1); the output P bound as [H, S, S] over storage [S, H, S].
    The batch stride (D) is below one batch's row span (S*H*D), so TMA tiles are
    refused and the gather loader / direct stores must give the exact result."""
    torch = _torch()
    h, s, d = 6, 96, 64
    rng = port.Rng(81)
    q = rng.tensor((h, s, d), True)
    k = rng.tensor((h, s, d), True)
    dag = batched_matmul_scale_dag(h, s, s, d, 0.125, DType.F32, "bnk")

    def interleaved(a):
        st = torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2), dtype=np.float32)).to(torch.bfloat16).cuda()
        return st.as_strided((h, s, d), (d, h * d, 1))

    qv, kv = interleaved(q), interleaved(k)
    out_store = torch.full((s, h, s), float("nan"), dtype=torch.float32, device="cuda")
    out = out_store.as_strided((h, s, s), (s, h * s, 1))
    for cfg in (ScheduleConfig(), ScheduleConfig(block_n=64, split_k=2), ScheduleConfig(block_m=256, block_n=128)):
        out_store.fill_(float("nan"))
        Plan(dag, cfg).bind([qv, kv], [out]).launch()
        torch.cuda.synchronize()
        want = port.batched_matmul_scale(q, k.transpose(0, 2, 1), 0.125)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), want)


def _f16(a):
    return np.asarray(a, np.float64).astype(np.float16).astype(np.float64)


@pytest.mark.parametrize("bm,bn,sk", [(128, 128, 1), (128, 256, 2), (256, 128, 1), (256, 256, 2), (128, 64, 4)])
@pytest.mark.parametrize("b_layout", [None, "t"])  # B[K,N] MN-major (TMA MN) / K-major
def test_fp16_matmul_exact(bm, bn, sk, b_layout):
    m, n, k = 520, 384, 448
    rng = port.Rng(82)
    a, b, bias = rng.tensor((m, k), True), rng.tensor((k, n), True), rng.tensor((n,), True)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, plan = run(dag, {"A": dev(a, "f16"), "B": dev(b, "f16", layout=b_layout), "Bias": dev(bias, "f32")},
                    {"D": (m, n)}, cfg=ScheduleConfig(block_m=bm, block_n=bn, split_k=sk))
    assert np.array_equal(got["D"], port.matmul_bias_relu(a, b, bias))


def test_fp16_matmul_float_tolerance():
    """fp16 values keep 11 significant bits: a bf16 reinterpretation (the round-1
    defect) or a silent bf16 down-conversion would fail this 1e-4 bound."""
    m, n, k = 512, 512, 512
    rng = port.Rng(83)
    a, b, bias = _f16(rng.tensor((m, k))), _f16(rng.tensor((k, n))), rng.tensor((n,))
    dag = matmul_epilogue_dag(m, n, k)
    for layout in (None, "t"):
        got, _ = run(dag, {"A": dev(a, "f16"), "B": dev(b, "f16", layout=layout), "Bias": dev(bias, "f32")},
                     {"D": (m, n)})
        assert port.max_rel_error(got["D"], port.matmul_bias_relu(a, b, bias)) <= 1e-4


def test_fp16_output_and_gather_operand():
    """fp16 output (direct stores) and an fp16 operand TMA cannot describe (odd row
    stride -> predicated gather, kept in fp16 format)."""
    torch = _torch()
    m, n, k = 200, 136, 77
    rng = port.Rng(84)
    a, b, bias = rng.tensor((m, k), True), rng.tensor((k, n), True), rng.tensor((n,), True)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a, "f16"), "B": dev(b, "f16"), "Bias": dev(bias, "f16")}, {"D": (m, n)},
                 out_dtype="f16")
    assert np.array_equal(got["D"], _f16(port.matmul_bias_relu(a, b, bias)))


@pytest.mark.parametrize("bm", [128, 256])
def test_fp16_conv_channels_last_exact(bm):
    n, c, h, w, f, kk, s, p = 2, 64, 10, 10, 128, 3, 1, 1
    rng = port.Rng(85)
    x, wt = rng.tensor((n, c, h, w), True), rng.tensor((f, c, kk, kk), True)
    scale, shift = rng.tensor((f,), True), rng.tensor((f,), True)
    dag = conv_bn_relu_dag(n, c, h, w, f, kk, kk, s, p, DType.I32)
    got, _ = run(dag, {"X": dev(x, "f16", "cl"), "W": dev(wt, "f16", "cl"), "Scale": dev(scale, "f32"),
                       "Shift": dev(shift, "f32")}, {"Z": (n, f, h, w)}, cfg=ScheduleConfig(block_m=bm))
    assert np.array_equal(got["Z"], port.conv_bn_relu(x, wt, scale, shift, s, p))


def test_mixed_bf16_fp16_operands_are_refused():
    m = n = k = 64
    rng = port.Rng(86)
    a, b, bias = rng.tensor((m, k), True), rng.tensor((k, n), True), rng.tensor((n,), True)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    with pytest.raises(TaskmapError) as e:
        run(dag, {"A": dev(a, "bf16"), "B": dev(b, "f16"), "Bias": dev(bias, "f32")}, {"D": (m, n)})
    assert e.value.status == 4


def _fig11_dag(n_rows=100, k=64, n=96, dtype=DType.F32):
    """SPEC.md:370-387 / PAPER.md:606 Fig. 11 on the GEMM anchor: the prologue
    A[i, k] = C[99 - i, k] * 2.0 (reversed re-index + arithmetic) feeds
    B = A W; the epilogue D[i / 50, i % 50, j] = B[i, j] * 3.0 (reshape-split remap)."""
    from paper_2210_09603_b200 import Axis, ComputeDAG, TensorNode, fimm, imm, load, mul, sub, var
    d = ComputeDAG()
    d.add_input("C", [n_rows, k], dtype)
    d.add_input("W", [k, n], dtype)
    d.add_compute("A", [Axis("i", n_rows), Axis("k", k)],
                  mul(load("C", [sub(imm(n_rows - 1), var("i")), var("k")]), fimm(2.0)), dtype)
    d.nodes.append(TensorNode("B", [n_rows, n], dtype, "reduce", [Axis("i", n_rows), Axis("j", n)], [Axis("kk", k)],
                              value=mul(load("A", [var("i"), var("kk")]), load("W", [var("kk"), var("j")]))))
    d.add_compute("D", [Axis("a", n_rows // 50), Axis("b", 50), Axis("j", n)],
                  mul(load("B", [add_(mul(var("a"), imm(50)), var("b")), var("j")]), fimm(3.0)), dtype)
    d.outputs = ["D"]
    return d


def add_(a, b):
    from paper_2210_09603_b200 import add
    return add(a, b)


@pytest.mark.parametrize("cfg", [ScheduleConfig(), ScheduleConfig(block_n=64, split_k=2),
                                 ScheduleConfig(block_m=256, block_n=128), ScheduleConfig(math="fp32_simt")])
def test_fig11_arithmetic_prologue_and_remap_epilogue(cfg):
    """Fig. 11 end to end on the GPU: one fused kernel whose gather loader reads
    C[99 - i, k] * 2.0 and whose epilogue stores B * 3.0 at (i / 50, i % 50);
    exact against reference_eval on integer data."""
    from gpu_util import have_ref, oracle_eval
    dag = _fig11_dag()
    rng = port.Rng(87)
    c, w = rng.tensor((100, 64), True), rng.tensor((64, 96), True)
    dt = "f32" if cfg.math == "fp32_simt" else "bf16"
    got, plan = run(dag, {"C": dev(c, dt), "W": dev(w, dt)}, {"D": (2, 50, 96)}, cfg=cfg)
    k0 = plan.describe()["kernels"][0]
    assert len(plan.describe()["kernels"]) == 1 and k0["prologue"] == ["A"] and k0["epilogue"] == ["D"]
    assert "C[99 - __row" in k0["A"] or "C[" in k0["A"]
    want = (3.0 * ((2.0 * c[::-1]) @ w)).reshape(2, 50, 96)
    assert np.array_equal(got["D"], want)
    if have_ref():
        assert np.array_equal(got["D"], oracle_eval(dag, {"C": c, "W": w}, {"D": (2, 50, 96)})["D"])


def test_relu_prologue_two_matmuls():
    """ReLU -> matmul -> matmul partitions into two kernels and the ReLU
    fuses into the first matmul's prologue only."""
    from paper_2210_09603_b200 import Axis, ComputeDAG, TensorNode, load, relu, var, mul
    m, k1, k2, n = 192, 96, 160, 128
    d = ComputeDAG()
    d.add_input("X", [m, k1], DType.I32)
    d.add_input("W1", [k1, k2], DType.I32)
    d.add_input("W2", [k2, n], DType.I32)
    d.add_compute("R", [Axis("i", m), Axis("k", k1)], relu(load("X", [var("i"), var("k")])), DType.I32)
    d.nodes.append(TensorNode("H", [m, k2], DType.I32, "reduce", [Axis("i", m), Axis("j", k2)], [Axis("k", k1)],
                              value=mul(load("R", [var("i"), var("k")]), load("W1", [var("k"), var("j")]))))
    d.nodes.append(TensorNode("Y", [m, n], DType.I32, "reduce", [Axis("i", m), Axis("j", n)], [Axis("k", k2)],
                              value=mul(load("H", [var("i"), var("k")]), load("W2", [var("k"), var("j")]))))
    d.outputs = ["Y"]
    rng = port.Rng(88)
    x, w1, w2 = rng.tensor((m, k1), True), rng.tensor((k1, k2), True), rng.tensor((k2, n), True)
    got, plan = run(d, {"X": dev(x, "f32"), "W1": dev(w1, "f32"), "W2": dev(w2, "f32")}, {"Y": (m, n)},
                    cfg=ScheduleConfig(math="tf32"))
    ks = plan.describe()["kernels"]
    assert len(ks) == 2 and ks[0]["prologue"] == ["R"] and ks[1]["prologue"] == []
    assert np.array_equal(got["Y"], (np.maximum(x, 0) @ w1) @ w2)
