"""Halo implicit-GEMM conv (conv_halo.cuh) against the oracle: stride-1 convs
with C % 64 == 0 on channels-last data (the ResNet-50 3x3 layers) stage one
channel-group-major input band per tile and read it from every tap's MMA at a
descriptor offset (the reference im2col node, proj/src/compute_ir.cpp:532-557,
never materialised).  Bit-exact on the reference's integer test data.
"""
import numpy as np
import pytest

from oracle import port
from paper_2210_09603_b200 import Plan, ScheduleConfig, workloads as W

pytestmark = pytest.mark.gpu
LD_HALO = 9


def _run(n, c, h, f, k, p, seed, expect_halo=True, cfg=None):
    import torch
    L = W.ConvLayer("t", c, h, f, k, 1, p, 1)
    rng = port.Rng(seed)
    x = rng.tensor((n, c, h, h), True)
    wt = rng.tensor((f, c, k, k), True)
    scale, shift = rng.tensor((f,), True), rng.tensor((f,), True)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()  # noqa: E731
    ho = L.out_hw()
    z = torch.full((n, f, ho, ho), float("nan"), dtype=torch.bfloat16, device="cuda").contiguous(
        memory_format=torch.channels_last)
    ins = [bf(x).contiguous(memory_format=torch.channels_last), bf(wt).contiguous(memory_format=torch.channels_last),
           torch.from_numpy(scale.astype(np.float32)).cuda(), torch.from_numpy(shift.astype(np.float32)).cuda()]
    ex = Plan(W.conv_bn_relu_dag(L, n), cfg or ScheduleConfig(math="halo")).bind(ins, [z])
    info = ex.kernel_info(0)
    assert (info["a_loader"] == LD_HALO) == expect_halo, info
    ex.launch()
    torch.cuda.synchronize()
    want = port.round_bf16(port.conv_bn_relu(x, wt, scale, shift, 1, p))
    return z.float().cpu().numpy().astype(np.float64), want


@pytest.mark.parametrize("n,c,h,f", [(1, 64, 56, 64), (1, 128, 28, 128), (2, 256, 14, 256), (1, 256, 28, 512)])
def test_halo_resnet_3x3_geometries_exact(n, c, h, f):
    got, want = _run(n, c, h, f, 3, 1, seed=400 + c)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,c,h,f,k,p", [(2, 64, 20, 128, 3, 1), (1, 64, 17, 64, 5, 2), (1, 64, 126, 64, 3, 1), (2, 192, 12, 192, 3, 1)])
def test_halo_ragged_shapes_exact(n, c, h, f, k, p):
    got, want = _run(n, c, h, f, k, p, seed=410 + h)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,c,h,f", [(1, 64, 130, 64), (2, 512, 7, 512), (3, 128, 9, 64), (1, 512, 14, 128)])
def test_halo_ineligible_falls_back(n, c, h, f):
    """The K3 (im2col) kernel runs when W + 2 pad > 128 pixels, when fewer than 96
    of the 128 TMEM lanes would hold output pixels (7x7 / 9x9 maps), or when two
    bands do not fit in shared memory (512 channels x 10 rows x 16 pixels)."""
    got, want = _run(n, c, h, f, 3, 1, seed=420 + h, expect_halo=False)
    assert np.array_equal(got, want)


def test_halo_only_when_scheduled():
    """The halo family is a point of schedule_space('conv2d'): other configs run K3."""
    got, want = _run(1, 64, 20, 64, 3, 1, seed=430, expect_halo=False, cfg=ScheduleConfig())
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,c,h,f,k,p", [(1, 64, 56, 64, 3, 1), (3, 128, 28, 128, 3, 1), (2, 256, 14, 256, 3, 1),
                                         (1, 64, 17, 64, 5, 2), (2, 192, 12, 192, 3, 1)])
def test_halo_cluster_pair_multicast_exact(monkeypatch, n, c, h, f, k, p):
    """TMB_HALO_MC=2: CTA pairs (clusters of 2) walk the same filter stages, each
    TMA-multicasting half of every stage (half the taps when a stage holds an even
    number, else half the filter rows) into both CTAs, with the MMA commits releasing
    the stage in both; an odd spatial tile count leaves the last pair's second CTA a
    duplicate tile that stores nothing."""
    monkeypatch.setenv("TMB_HALO_MC", "2")
    got, want = _run(n, c, h, f, k, p, seed=430 + c + h)
    assert np.array_equal(got, want)
