"""Parity at the large shapes bench.py's `large_shapes` line measures (the north-star
>= 70% target): the 8192^3 matmul + bias + ReLU and the ResNet-50 3x3 conv + BN + ReLU
layers at batch 256, with the CTA-pair (256 x 256) and single-CTA (128 x 256)
schedules that line picks from.

The CPU oracle cannot evaluate these sizes in seconds, so the check is a
size-independent property: on integer-valued inputs small enough that every
product and every fp32 partial sum is exact, the fused kernel's bf16 output must
equal round_bf16 of the exact result.  The exact result is computed in float64 on
the device for sampled rows / images (test-only reference; the product never calls
torch math)."""
import pytest

from paper_2210_09603_b200 import Plan, ScheduleConfig, workloads as W

pytestmark = pytest.mark.gpu


def _ints(torch, shape, lo, hi, gen, dtype):
    return torch.randint(lo, hi + 1, shape, generator=gen, device="cuda").to(dtype)


@pytest.mark.parametrize("bm,bn", [(256, 256), (128, 256)])
def test_gemm_8192_bias_relu_exact(bm, bn):
    import torch
    m = n = k = 8192
    g = torch.Generator(device="cuda")
    g.manual_seed(bm + bn)
    a = _ints(torch, (m, k), -2, 2, g, torch.bfloat16)
    b = _ints(torch, (k, n), -2, 2, g, torch.bfloat16)
    bias = _ints(torch, (n,), -64, 64, g, torch.float32)
    d = torch.full((m, n), float("nan"), device="cuda", dtype=torch.bfloat16)
    Plan(W.matmul_bias_relu_dag(m, n, k), ScheduleConfig(block_m=bm, block_n=bn)).bind([a, b, bias], [d]).launch()
    torch.cuda.synchronize()
    rows = torch.cat([torch.arange(0, 128, device="cuda"), torch.randint(128, m, (128,), generator=g, device="cuda"),
                      torch.arange(m - 128, m, device="cuda")])
    want = torch.relu(a[rows].double() @ b.double() + bias.double()).to(torch.bfloat16)
    got = d[rows]
    assert torch.equal(got, want), (got.float() - want.float()).abs().max().item()


@pytest.mark.parametrize("lname,bm,bn", [("l3.c2", 256, 256), ("l3.c2", 128, 256), ("l4.c2", 256, 256)])
def test_conv_batch256_bn_relu_exact(lname, bm, bn):
    import torch
    L = next(x for x in W.RESNET50 if x.name == lname)
    B = 256
    g = torch.Generator(device="cuda")
    g.manual_seed(7 + bm)
    fmt = torch.channels_last
    x = _ints(torch, (B, L.c, L.h, L.h), -2, 2, g, torch.bfloat16).contiguous(memory_format=fmt)
    w = _ints(torch, (L.f, L.c, L.k, L.k), -2, 2, g, torch.bfloat16).contiguous(memory_format=fmt)
    scale = _ints(torch, (L.f,), -3, 3, g, torch.float32)
    shift = _ints(torch, (L.f,), -64, 64, g, torch.float32)
    ho = L.out_hw()
    o = torch.full((B, L.f, ho, ho), float("nan"), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=fmt)
    ex = Plan(W.conv_bn_relu_dag(L, B), ScheduleConfig(block_m=bm, block_n=bn)).bind([x, w, scale, shift], [o])
    ex.launch()
    torch.cuda.synchronize()
    imgs = torch.tensor([0, 1, 97, 128, 200, 255], device="cuda")
    acc = torch.nn.functional.conv2d(x[imgs].double(), w.double(), stride=L.s, padding=L.p)
    want = torch.relu(acc * scale.double().view(1, -1, 1, 1) + shift.double().view(1, -1, 1, 1)).to(torch.bfloat16)
    got = o[imgs]
    assert torch.equal(got, want), (got.float() - want.float()).abs().max().item()
