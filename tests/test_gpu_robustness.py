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
