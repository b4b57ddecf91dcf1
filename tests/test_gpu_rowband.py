"""Row-band implicit-GEMM conv (conv_rowband.cuh) against the oracle.

Small-C convolutions whose input pixels are padded to 4 channels (8-byte pixels,
stride 2 -- the ResNet-50 stem conv1) or 8 channels (16-byte pixels, stride 1)
run the row-band kernel: the MMA reads its A operand straight out of staged
input rows (reference im2col node, proj/src/compute_ir.cpp:532-557, never
materialised).  Compared with the oracle port (pinned to reference_eval by
tests/golden) on the reference's integer test data: bit-exact.
"""
import numpy as np
import pytest

from oracle import port
from paper_2210_09603_b200 import Plan, ScheduleConfig, workloads as W

pytestmark = pytest.mark.gpu
LD_ROWBAND = 8


def _torch():
    import torch
    return torch


def _bf16(a):
    t = _torch()
    return t.from_numpy(np.ascontiguousarray(a, np.float32)).to(t.bfloat16).cuda()


def _padded_x(x, cpad, pad_value=0.0):
    """X[n,c,h,w] stored channels-last with each pixel padded to cpad channels."""
    torch = _torch()
    n, c, h, w = x.shape
    xb = torch.full((n, h, w, cpad), pad_value, dtype=torch.bfloat16, device="cuda")
    xb[..., :c] = _bf16(x).permute(0, 2, 3, 1)
    return xb.as_strided((n, c, h, w), (h * w * cpad, 1, w * cpad, cpad))


def _run(n, c, h, f, k, s, p, cpad, seed, pad_value=0.0, expect_rowband=True):
    torch = _torch()
    L = W.ConvLayer("t", c, h, f, k, s, p, 1)
    rng = port.Rng(seed)
    x = rng.tensor((n, c, h, h), True)
    wt = rng.tensor((f, c, k, k), True)
    scale, shift = rng.tensor((f,), True), rng.tensor((f,), True)
    ho = L.out_hw()
    z = torch.full((n, f, ho, ho), float("nan"), dtype=torch.bfloat16, device="cuda").contiguous(
        memory_format=torch.channels_last)
    ins = [_padded_x(x, cpad, pad_value), _bf16(wt).contiguous(memory_format=torch.channels_last),
           torch.from_numpy(scale.astype(np.float32)).cuda(), torch.from_numpy(shift.astype(np.float32)).cuda()]
    ex = Plan(W.conv_bn_relu_dag(L, n), ScheduleConfig(block_n=64)).bind(ins, [z])
    info = ex.kernel_info(0)
    assert (info["a_loader"] == LD_ROWBAND) == expect_rowband, info
    ex.launch()
    torch.cuda.synchronize()
    want = port.round_bf16(port.conv_bn_relu(x, wt, scale, shift, s, p))
    return z.float().cpu().numpy().astype(np.float64), want


def test_rowband_conv1_geometry_exact():
    """ResNet-50 conv1 (3 -> 64, 7x7, stride 2, pad 3) on 224x224, NHWC4 input."""
    got, want = _run(1, 3, 224, 64, 7, 2, 3, cpad=4, seed=301)
    assert np.array_equal(got, want)


def test_rowband_conv1_two_images_band_crossing():
    """Bands never cross images; 2 images x 112 rows over the persistent grid."""
    got, want = _run(2, 3, 224, 64, 7, 2, 3, cpad=4, seed=302)
    assert np.array_equal(got, want)


def test_rowband_pad_lanes_with_nan_are_ignored():
    """The caller's padding channel holds NaN: staged pad lanes are zeroed."""
    got, want = _run(1, 3, 64, 64, 7, 2, 3, cpad=4, seed=303, pad_value=float("nan"))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("h,f,k,p", [(34, 64, 7, 3), (18, 32, 5, 2), (40, 128, 3, 1), (10, 64, 1, 0), (66, 200, 7, 3)])
def test_rowband_stride2_ragged_shapes(h, f, k, p):
    got, want = _run(2, 3, h, f, k, 2, p, cpad=4, seed=304 + h)
    assert np.array_equal(got, want)


def test_rowband_odd_width_nhwc4_falls_back():
    """An odd row of 8-byte pixels is not a whole number of 16-byte granules."""
    got, want = _run(1, 3, 33, 64, 7, 2, 3, cpad=4, seed=335, expect_rowband=False)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("c,h,f,k,p", [(3, 20, 64, 3, 1), (8, 31, 96, 5, 2), (5, 128, 64, 7, 3), (1, 12, 256, 3, 0)])
def test_rowband_stride1_nhwc8(c, h, f, k, p):
    got, want = _run(2, c, h, f, k, 1, p, cpad=8, seed=320 + c + h)
    assert np.array_equal(got, want)


def test_rowband_ineligible_falls_back():
    """Wo > 128 (one tile per output row cannot hold it): the K3 kernel runs."""
    got, want = _run(1, 3, 300, 64, 3, 2, 1, cpad=4, seed=330, expect_rowband=False)
    assert np.array_equal(got, want)
