"""GPU parity of the fused tcgen05 GEMM path against the reference oracle.

Exact cases use the reference's i32 test data U{-8..8} (tensor.cpp:66), which
is exact in bf16, with fp32 accumulation and fp32 output: the device result
must equal reference_eval bit for bit.  Float cases feed the
same bf16/tf32-rounded values to both sides; tolerance max_rel_error <= 1e-4
for fp32 outputs, 1e-2 for bf16 outputs, 2e-2 for the FFN chain
whose bf16 intermediate H the fp64 oracle cannot model.
"""
import numpy as np
import pytest

from oracle import port
from paper_2210_09603_b200 import DType, ScheduleConfig

from dags import batched_matmul_scale_dag, conv_bn_relu_dag, ffn_dag, matmul_epilogue_dag
from gpu_util import dev, have_ref, oracle_eval, rounded, run

pytestmark = pytest.mark.gpu


def _matmul_case(m, n, k, exact, seed):
    rng = port.Rng(seed)
    a = rng.tensor((m, k), exact)
    b = rng.tensor((k, n), exact)
    bias = rng.tensor((n,), exact)
    if not exact:
        a, b, bias = rounded(a, "bf16"), rounded(b, "bf16"), rounded(bias, "f32")
    return a, b, bias


@pytest.mark.parametrize("bm,bn", [(128, 64), (128, 96), (128, 128), (128, 192), (128, 256), (256, 64), (256, 128),
                                   (256, 256)])
@pytest.mark.parametrize("b_layout", [None, "t"])  # B[K,N] MN-major (TMA MN) / K-major storage
def test_matmul_bias_relu_exact(bm, bn, b_layout):
    """block_m=256 runs the SM-pair form (tcgen05.mma.cta_group::2)."""
    m, n, k = 640, 320, 192
    a, b, bias = _matmul_case(m, n, k, True, 2)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a), "B": dev(b, layout=b_layout), "Bias": dev(bias, "f32")}, {"D": (m, n)},
                 cfg=ScheduleConfig(block_m=bm, block_n=bn))
    want = oracle_eval(dag, {"A": a, "B": b, "Bias": bias}, {"D": (m, n)}) if have_ref() else \
        {"D": port.matmul_bias_relu(a, b, bias)}
    assert np.array_equal(got["D"], want["D"])


@pytest.mark.parametrize("pipeline", [True, False])
@pytest.mark.parametrize("raster", [0, 1])
@pytest.mark.parametrize("split_k", [1, 3])
def test_matmul_schedule_variants_bit_identical(pipeline, raster, split_k):
    """pipeline on/off and split-K are bit-identical on i32 data."""
    m, n, k = 384, 256, 320
    a, b, bias = _matmul_case(m, n, k, True, 7)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias, "f32")}, {"D": (m, n)},
                 cfg=ScheduleConfig(pipeline=pipeline, stages=0 if pipeline else 2, raster=raster, split_k=split_k))
    assert np.array_equal(got["D"], port.matmul_bias_relu(a, b, bias))


@pytest.mark.parametrize("bm,bn,split_k", [(128, 128, 2), (256, 256, 4), (256, 128, 5), (128, 64, 8)])
def test_split_k_repeat_launch_deterministic(bm, bn, split_k):
    """Split-K with self-resetting tile counters: repeated launches give identical results."""
    import torch
    from paper_2210_09603_b200 import Plan
    m, n, k = 520, 384, 1000
    rng = port.Rng(31)
    a, b = rounded(rng.tensor((m, k)), "bf16"), rounded(rng.tensor((k, n)), "bf16")
    bias = rng.tensor((n,))
    dag = matmul_epilogue_dag(m, n, k)
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    ex = Plan(dag, ScheduleConfig(block_m=bm, block_n=bn, split_k=split_k)).bind(
        [dev(a), dev(b), dev(bias, "f32")], [out])
    results = []
    for _ in range(3):
        out.fill_(float("nan"))
        ex.launch()
        torch.cuda.synchronize()
        results.append(out.cpu().numpy().copy())
    assert all(np.array_equal(results[0], r) for r in results[1:])
    assert port.max_rel_error(results[0], port.matmul_bias_relu(a, b, bias)) <= 1e-4


def test_matmul_float_tolerance():
    m = n = k = 1024
    a, b, bias = _matmul_case(m, n, k, False, 1)
    dag = matmul_epilogue_dag(m, n, k)
    got, _ = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias, "f32")}, {"D": (m, n)})
    assert port.max_rel_error(got["D"], port.matmul_bias_relu(a, b, bias)) <= 1e-4


def test_matmul_float_vs_reference_eval_small():
    m, n, k = 128, 128, 128
    a, b, bias = _matmul_case(m, n, k, False, 11)
    dag = matmul_epilogue_dag(m, n, k)
    got, _ = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias, "f32")}, {"D": (m, n)})
    if not have_ref():
        pytest.skip("reference library not built")
    want = oracle_eval(dag, {"A": a, "B": b, "Bias": bias}, {"D": (m, n)})
    assert port.max_rel_error(got["D"], want["D"]) <= 1e-4


def test_matmul_bf16_output():
    m, n, k = 512, 512, 256
    a, b, bias = _matmul_case(m, n, k, False, 3)
    dag = matmul_epilogue_dag(m, n, k)
    got, _ = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias)}, {"D": (m, n)}, out_dtype="bf16")
    assert port.max_rel_error(got["D"], port.matmul_bias_relu(a, b, rounded(bias, "bf16"))) <= 1e-2


@pytest.mark.parametrize("bm,bn", [(128, 64), (128, 96), (128, 128), (128, 192), (128, 256), (256, 64), (256, 128),
                                   (256, 256)])
@pytest.mark.parametrize("mn", [(333, 200), (640, 520)])
def test_lean_drain_bf16_output_exact(bm, bn, mn):
    """bf16 TMA-stored output + canonical epilogue: the lean drain path, the two
    epilogue warp groups each draining one column half of every tile (ragged M/N:
    half tiles that are partly or wholly outside N).  Integer data keeps every
    fp32 intermediate exact, so the device must equal round_bf16(reference)."""
    m, n = mn
    k = 320
    a, b, bias = _matmul_case(m, n, k, True, 41)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias, "f32")}, {"D": (m, n)}, out_dtype="bf16",
                 cfg=ScheduleConfig(block_m=bm, block_n=bn))
    assert np.array_equal(got["D"], port.round_bf16(port.matmul_bias_relu(a, b, bias)))


@pytest.mark.parametrize("bm,bn,split_k", [(128, 128, 2), (128, 256, 3), (256, 128, 2), (128, 64, 4), (128, 192, 3),
                                           (128, 96, 2)])
def test_lean_split_k_bf16_exact(bm, bn, split_k):
    """Split-K with the lean drain: each epilogue group parks its column half of the
    partial tile, the last arriver of each (tile, half) reduces in split order and
    stores bf16; repeated launches reuse the self-resetting counters."""
    import torch
    from paper_2210_09603_b200 import Plan
    m, n, k = 520, 328, 1000
    a, b, bias = _matmul_case(m, n, k, True, 45)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    out = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    ex = Plan(dag, ScheduleConfig(block_m=bm, block_n=bn, split_k=split_k)).bind(
        [dev(a), dev(b), dev(bias, "f32")], [out])
    assert ex.kernel_info(0)["split_k"] == split_k
    want = port.round_bf16(port.matmul_bias_relu(a, b, bias))
    for _ in range(3):
        out.fill_(float("nan"))
        ex.launch()
        torch.cuda.synchronize()
        assert np.array_equal(out.float().cpu().numpy().astype(np.float64), want)


@pytest.mark.parametrize("bn", [128, 256])
def test_lean_drain_residual_exact(bn):
    """D = relu(A B + bias) + R with a bf16 residual (the FFN's second GEMM form)."""
    import torch
    from paper_2210_09603_b200 import Axis, Plan, add, load, relu, var
    from paper_2210_09603_b200 import matmul_dag
    m, n, k = 384, 320, 256
    a, b, bias = _matmul_case(m, n, k, True, 43)
    r = port.Rng(44).tensor((m, n), True)
    dag = matmul_dag(m, n, k, DType.I32)
    dag.add_input("Bias", [n], DType.I32)
    dag.add_input("R", [m, n], DType.I32)
    dag.add_compute("D", [Axis("i", m), Axis("j", n)],
                    add(relu(add(load("C", [var("i"), var("j")]), load("Bias", [var("j")]))),
                        load("R", [var("i"), var("j")])), DType.I32)
    dag.outputs = ["D"]
    out = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
    Plan(dag, ScheduleConfig(block_n=bn)).bind([dev(a), dev(b), dev(bias, "f32"), dev(r)], [out]).launch()
    torch.cuda.synchronize()
    want = port.round_bf16(port.matmul_bias_relu(a, b, bias) + r)
    assert np.array_equal(out.float().cpu().numpy().astype(np.float64), want)


@pytest.mark.parametrize("mnk", [(2039, 2039, 2039), (1, 1, 1), (130, 17, 5), (7, 300, 77)])
def test_matmul_prime_and_tiny_sizes(mnk):
    """any M,N,K >= 1 (2039^3 is where input-centric spaces fail)."""
    m, n, k = mnk
    a, b, bias = _matmul_case(m, n, k, True, 5)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias, "f32")}, {"D": (m, n)})
    assert np.array_equal(got["D"], port.matmul_bias_relu(a, b, bias))


def test_matmul_gelu_epilogue():
    m, n, k = 256, 512, 256
    a, b, bias = _matmul_case(m, n, k, False, 9)
    dag = matmul_epilogue_dag(m, n, k, act="gelu")
    got, plan = run(dag, {"A": dev(a), "B": dev(b), "Bias": dev(bias, "f32")}, {"D": (m, n)})
    assert [o["kind"] for o in plan.describe()["kernels"][0]["ops"]] == [16, 33]  # ADD_T, GELU_TANH
    want = port.gelu_tanh(port.matmul(a, b) + bias[None, :])
    assert port.max_rel_error(got["D"], want) <= 1e-4


def test_fp32_config1_cuda_core_path():
    """config 1: fp32 matmul M=N=K=1024 + bias + ReLU, unrounded U(-1,1) fp32 inputs, on the
    task-mapped CUDA-core kernel (math auto -> fp32_simt): max_rel_error <= 1e-4."""
    m = n = k = 1024
    rng = port.Rng(1)
    a, b, bias = rounded(rng.tensor((m, k)), "f32"), rounded(rng.tensor((k, n)), "f32"), rounded(rng.tensor((n,)), "f32")
    dag = matmul_epilogue_dag(m, n, k)
    got, plan = run(dag, {"A": dev(a, "f32"), "B": dev(b, "f32"), "Bias": dev(bias, "f32")}, {"D": (m, n)})
    assert port.max_rel_error(got["D"], port.matmul_bias_relu(a, b, bias)) <= 1e-4


@pytest.mark.parametrize("mnk", [(256, 256, 256), (2039, 67, 131), (1, 1, 1)])
def test_fp32_cuda_core_exact_int(mnk):
    m, n, k = mnk
    a, b, bias = _matmul_case(m, n, k, True, 8)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a, "f32"), "B": dev(b, "f32"), "Bias": dev(bias, "f32")}, {"D": (m, n)},
                 cfg=ScheduleConfig(math="fp32_simt"))
    want = oracle_eval(dag, {"A": a, "B": b, "Bias": bias}, {"D": (m, n)}) if (have_ref() and m * n * k < 2e7) \
        else {"D": port.matmul_bias_relu(a, b, bias)}
    assert np.array_equal(got["D"], want["D"])


@pytest.mark.parametrize("mnk,bn,bk", [((256, 256, 256), 64, 8), ((2039, 67, 131), 64, 16), ((1024, 1024, 1024), 64, 16),
                                       ((300, 200, 77), 128, 16), ((129, 130, 15), 128, 8)])
def test_fp32_cuda_core_tile_variants_exact_int(mnk, bn, bk):
    """The 128x64 CUDA-core tile (spatial(4,2)*repeat(2,1)*spatial(4,8)*repeat(4,4)) and ragged edges."""
    m, n, k = mnk
    a, b, bias = _matmul_case(m, n, k, True, 81)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    got, _ = run(dag, {"A": dev(a, "f32"), "B": dev(b, "f32"), "Bias": dev(bias, "f32")}, {"D": (m, n)},
                 cfg=ScheduleConfig(math="fp32_simt", block_n=bn, block_k=bk))
    assert np.array_equal(got["D"], port.matmul_bias_relu(a, b, bias))


@pytest.mark.parametrize("bn,sk", [(128, 1), (256, 2)])
def test_matmul_tf32_row_major_b(bn, sk):
    """kind::tf32 with B [K,N] row-major: MN-major fp32 B TMA-fed in the 32-byte-atom 128-byte
    swizzle (UMMA layout SWIZZLE_128B_BASE32B, the only MN-major layout kind::tf32 takes)."""
    m, n, k = 512, 384, 256
    rng = port.Rng(13)
    a, b = rounded(rng.tensor((m, k)), "tf32"), rounded(rng.tensor((k, n)), "tf32")
    bias = rounded(rng.tensor((n,)), "f32")
    dag = matmul_epilogue_dag(m, n, k)
    got, _ = run(dag, {"A": dev(a, "f32"), "B": dev(b, "f32"), "Bias": dev(bias, "f32")}, {"D": (m, n)},
                 cfg=ScheduleConfig(math="tf32", block_n=bn, split_k=sk))
    assert port.max_rel_error(got["D"], port.matmul_bias_relu(a, b, bias)) <= 1e-4


def test_matmul_tf32():
    m, n, k = 512, 384, 256
    rng = port.Rng(12)
    a, b = rounded(rng.tensor((m, k)), "tf32"), rounded(rng.tensor((k, n)), "tf32")
    bias = rounded(rng.tensor((n,)), "f32")
    dag = matmul_epilogue_dag(m, n, k)
    got, _ = run(dag, {"A": dev(a, "f32"), "B": dev(b, "f32", layout="t"), "Bias": dev(bias, "f32")}, {"D": (m, n)},
                 cfg=ScheduleConfig(math="tf32"))
    assert port.max_rel_error(got["D"], port.matmul_bias_relu(a, b, bias)) <= 1e-4


@pytest.mark.parametrize("kt_layout", ["bkn", "bnk"])
def test_batched_matmul_scale(kt_layout):
    b, m, n, k = 6, 128, 128, 64
    rng = port.Rng(3)
    q = rng.tensor((b, m, k), True)
    kt = rng.tensor((b, k, n), True)
    dag = batched_matmul_scale_dag(b, m, n, k, 0.125, DType.F32, kt_layout)
    kin = kt if kt_layout == "bkn" else np.ascontiguousarray(kt.transpose(0, 2, 1))
    name = "KT" if kt_layout == "bkn" else "Kmat"
    got, _ = run(dag, {"Q": dev(q), name: dev(kin)}, {"P": (b, m, n)})
    want = port.batched_matmul_scale(q, kt, 0.125)
    assert np.array_equal(got["P"], want)
    if have_ref():
        ref = oracle_eval(dag, {"Q": q, name: kin}, {"P": (b, m, n)})
        assert np.array_equal(got["P"], ref["P"])


@pytest.mark.parametrize("geom", [(2, 64, 8, 8, 64, 3, 3, 1, 1), (2, 64, 9, 9, 128, 3, 3, 2, 1),
                                  (2, 128, 7, 7, 64, 1, 1, 1, 0), (2, 64, 8, 8, 256, 1, 1, 2, 0),
                                  (1, 3, 20, 20, 64, 7, 7, 2, 3)])
@pytest.mark.parametrize("layout,bm", [(None, 128), ("cl", 128), ("cl", 256)])
def test_conv_bn_relu_exact(geom, layout, bm):
    """im2col prologue + BN-fold/ReLU + NCHW re-index epilogue, exact on i32 data."""
    n, c, h, w, f, kh, kw, s, p = geom
    rng = port.Rng(4)
    x = rng.tensor((n, c, h, w), True)
    wt = rng.tensor((f, c, kh, kw), True)
    scale = rng.tensor((f,), True)
    shift = rng.tensor((f,), True)
    dag = conv_bn_relu_dag(n, c, h, w, f, kh, kw, s, p, DType.I32)
    ho, wo = port.conv_out_extent(h, kh, s, p), port.conv_out_extent(w, kw, s, p)
    got, plan = run(dag, {"X": dev(x, layout=layout), "W": dev(wt, layout=layout), "Scale": dev(scale, "f32"),
                          "Shift": dev(shift, "f32")}, {"Z": (n, f, ho, wo)},
                    cfg=ScheduleConfig(block_m=bm, block_n=128 if bm == 256 else 128))
    want = port.conv_bn_relu(x, wt, scale, shift, s, p)
    assert np.array_equal(got["Z"], want)
    if have_ref() and n * f * ho * wo * c * kh * kw < 3e6:
        ref = oracle_eval(dag, {"X": x, "W": wt, "Scale": scale, "Shift": shift}, {"Z": (n, f, ho, wo)})
        assert np.array_equal(got["Z"], ref["Z"])


@pytest.mark.parametrize("geom", [(2, 3, 20, 20, 64, 7, 7, 2, 3), (1, 3, 17, 19, 32, 3, 3, 1, 1),
                                  (2, 4, 9, 9, 16, 5, 5, 2, 2)])
def test_conv_small_channel_g8_exact(geom):
    """conv1-style C <= 8 on 16-byte padded channels-last input: one 16-byte gather per
    (pixel, tap) (LD_IM2COL_G8, no-swizzle UMMA layout); pad channels are NaN in memory
    and must be masked, padding taps zero (compute_ir.cpp:539-553)."""
    n, c, h, w, f, kh, kw, s, p = geom
    rng = port.Rng(6)
    x = rng.tensor((n, c, h, w), True)
    wt = rng.tensor((f, c, kh, kw), True)
    scale, shift = rng.tensor((f,), True), rng.tensor((f,), True)
    dag = conv_bn_relu_dag(n, c, h, w, f, kh, kw, s, p, DType.I32)
    ho, wo = port.conv_out_extent(h, kh, s, p), port.conv_out_extent(w, kw, s, p)
    import torch
    from paper_2210_09603_b200 import Plan
    xs = dev(x, layout="cl8")
    out = torch.empty((n, f, ho, wo), dtype=torch.float32, device="cuda")
    ex = Plan(dag).bind([xs, dev(wt, layout="cl"), dev(scale, "f32"), dev(shift, "f32")], [out])
    assert ex.kernel_info(0)["a_loader"] == 7  # LD_IM2COL_G8
    ex.launch()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().astype(np.float64), port.conv_bn_relu(x, wt, scale, shift, s, p))


def test_conv_float_channels_last_output():
    """Float conv with the output bound channels-last (epilogue remap from the output's strides)."""
    import torch
    n, c, h, w, f, k, s, p = 4, 64, 14, 14, 128, 3, 1, 1
    rng = port.Rng(21)
    x, wt = rounded(rng.tensor((n, c, h, w)), "bf16"), rounded(rng.tensor((f, c, k, k)), "bf16")
    scale, shift = rng.tensor((f,)), rng.tensor((f,))
    dag = conv_bn_relu_dag(n, c, h, w, f, k, k, s, p)
    out = torch.empty((n, f, h, w), dtype=torch.float32, device="cuda").contiguous(memory_format=torch.channels_last)
    from paper_2210_09603_b200 import Plan
    Plan(dag).bind([dev(x, layout="cl"), dev(wt, layout="cl"), dev(scale, "f32"), dev(shift, "f32")], [out]).launch()
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    assert port.max_rel_error(got, port.conv_bn_relu(x, wt, scale, shift, s, p)) <= 1e-4


def test_ffn_chain():
    t, dm, dff = 256, 128, 512
    rng = port.Rng(5)
    x, w1, b1 = rounded(rng.tensor((t, dm)), "bf16"), rounded(rng.tensor((dm, dff)), "bf16"), rounded(rng.tensor((dff,)), "bf16")
    w2, b2 = rounded(rng.tensor((dff, dm)), "bf16"), rounded(rng.tensor((dm,)), "bf16")
    dag = ffn_dag(t, dm, dff)
    got, plan = run(dag, {"X": dev(x), "W1": dev(w1), "b1": dev(b1), "W2": dev(w2), "b2": dev(b2)}, {"O": (t, dm)},
                    out_dtype="bf16")
    assert len(plan.describe()["kernels"]) == 2
    # The device stores the intermediate H in bf16 (the fp64 oracle cannot
    # express that rounding, expr.hpp:16) and, because H is bf16, evaluates its
    # GELU with tanh.approx (rel. err 2^-11, below bf16's 2^-8 ulp). With the
    # bf16 rounding modelled, the remaining error is the bf16 output rounding
    # plus the accumulated tanh.approx error: max_rel_error <= 2e-2 (the bf16
    # chain tolerance of SURVEY.md §8c).
    assert port.max_rel_error(got["O"], port.ffn(x, w1, b1, w2, b2, round_h=port.round_bf16)) <= 2e-2
    # Unmodelled, the bf16(H) error (~2^-9 |H| per term, summed over dff) is an
    # absolute error, so bound it relative to the output scale.
    want = port.ffn(x, w1, b1, w2, b2)
    assert np.abs(got["O"] - want).max() / np.abs(want).max() <= 1e-2


def test_graph_replay_matches_eager_and_times_each_exec():
    """tm_graph: a captured sequence of execs (including a split-K one, whose
    counters must self-reset across replays) reproduces the eager results, and a
    timed graph reports one positive duration per exec."""
    import torch
    from paper_2210_09603_b200 import Graph, Plan
    m, n, k = 384, 256, 320
    a, b, bias = _matmul_case(m, n, k, True, 41)
    dag = matmul_epilogue_dag(m, n, k, DType.I32)
    ins = [dev(a), dev(b), dev(bias, "f32")]
    outs = [torch.empty((m, n), dtype=torch.float32, device="cuda") for _ in range(2)]
    execs = [Plan(dag, ScheduleConfig(split_k=sk)).bind(ins, [o]) for sk, o in zip((1, 3), outs)]
    want = port.matmul_bias_relu(a, b, bias)
    for timed in (False, True):
        g = Graph(execs, timed=timed)
        for _ in range(3):
            for o in outs:
                o.fill_(float("nan"))
            g.launch()
            torch.cuda.synchronize()
            for o in outs:
                assert np.array_equal(o.cpu().numpy(), want)
        if timed:
            ms = g.exec_ms()
            assert len(ms) == 2 and all(t > 0 for t in ms)
