"""ResNet-50 as one chain of the product's tensor programs:
the stage DAGs it adds (conv with the residual add fused into the epilogue, the
guarded max pool, the average pool, the classifier) against reference_eval on
small integer inputs (exact), every stage of the chain against the fp32 PyTorch
restatement (tests/chain_ref.py) from the chain's own inputs, the whole forward
against it end to end, and the CUDA-graph replay against eager launches."""
import numpy as np
import pytest

from chain_ref import chain_ref, stage_ref
from gpu_util import dev, have_ref, oracle_eval, run
from oracle import port
from paper_2210_09603_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _need_ref():
    if not have_ref():
        pytest.skip("reference library (oracle/_ref) not built")


def _exact(dag, inputs_np, out_shapes, dtype="bf16"):
    _need_ref()
    got, plan = run(dag, {k: dev(v, dtype) for k, v in inputs_np.items()}, out_shapes, "f32")
    want = oracle_eval(dag, inputs_np, out_shapes)
    for o in dag.outputs:
        assert np.array_equal(got[o], want[o]), o
    return plan


@pytest.mark.parametrize("relu_out,residual", [(True, True), (False, False)])
def test_conv_residual_and_downsample_epilogues_exact(relu_out, residual):
    """c3 (BN + residual + ReLU) and the downsample conv (BN only) on integer data."""
    L = W.ConvLayer("t", 32, 10, 64, 1, 1, 0, 1)
    d = W.conv_bn_dag(L, 2, relu_out=relu_out, residual=residual)
    rng = port.Rng(601)
    ins = {"X": rng.tensor((2, 32, 10, 10), True), "W": rng.tensor((64, 32, 1, 1), True),
           "Scale": rng.tensor((64,), True), "Shift": rng.tensor((64,), True)}
    if residual:
        ins["R"] = rng.tensor((2, 64, 10, 10), True)
    names = d.inputs
    assert set(names) == set(ins), names
    _exact(d, ins, {"Z": (2, 64, 10, 10)})


def test_maxpool_guarded_exact():
    d = W.maxpool_dag(2, 16, 13)
    ho = 7
    _exact(d, {"X": port.Rng(602).tensor((2, 16, 13, 13), True)}, {"Y": (2, 16, ho, ho)})


def test_avgpool_and_linear_against_oracle():
    _need_ref()
    d = W.avgpool_dag(2, 64, 7)
    x = port.Rng(603).tensor((2, 64, 7, 7))
    got, _ = run(d, {"X": dev(x, "f32")}, {"G": (2, 64)}, "f32")
    want = oracle_eval(d, {"X": x}, {"G": (2, 64)})
    assert port.max_rel_error(got["G"], want["G"]) <= 1e-5
    d = W.linear_dag(4, 40, 64)
    rng = port.Rng(604)
    ins = {"A": rng.tensor((4, 64), True), "B": rng.tensor((64, 40), True), "Bias": rng.tensor((40,), True)}
    _exact(d, ins, {"D": (4, 40)})


def _chain(batch, image, **kw):
    import torch
    from paper_2210_09603_b200.chain import ResNet50Chain
    c = ResNet50Chain(batch, image, **kw)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    c.set_input(torch.empty((batch, 3, image, image), device="cuda").uniform_(-1, 1, generator=g))
    return c


def _rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-6))


def test_chain_every_stage_against_fp32_reference():
    """Each stage recomputed in fp32 from the chain's own input activations:
    the only difference is accumulation order before the bf16 store (<= 2 bf16
    ulps of the stage's scale)."""
    import torch
    c = _chain(2, 64)
    assert [s.kind for s in c.stages].count("conv") == 53 and len(c.stages) == 56
    c.forward()
    torch.cuda.synchronize()
    acts = {k: v.float() for k, v in c.acts.items()}
    for st in c.stages:
        want = stage_ref(c, st, acts)
        assert _rel(acts[st.dst], want) <= 1.6e-2, (st.dst, _rel(acts[st.dst], want))


def test_chain_end_to_end_and_graph_replay():
    import torch
    c = _chain(4, 96)
    c.forward()
    torch.cuda.synchronize()
    eager = c.logits.clone()
    want = chain_ref(c)["logits"]
    assert torch.isfinite(eager).all()
    assert _rel(eager, want) <= 5e-2, _rel(eager, want)
    c.logits.zero_()
    c.replay()
    torch.cuda.synchronize()
    assert torch.equal(c.logits, eager)


def test_full_size_chain_batch32():
    """The configs[4] batch (32 images, 224^2) through all 53 convs in one graph."""
    import torch
    c = _chain(32, 224)
    c.replay()
    torch.cuda.synchronize()
    want = chain_ref(c)["logits"]
    assert _rel(c.logits, want) <= 5e-2, _rel(c.logits, want)
    assert c.flops > 1.3e11  # 4.1 GFLOP per image


@pytest.mark.parametrize("split_k", [1, 2, 4])
def test_residual_before_relu_compact_drain_exact(split_k):
    """The chain's c3 epilogue relu(acc*S + T + R) on the compact (TMA-fed,
    TMA-stored) kernel: channels-last bf16 in and out, integer data -> the fp32
    value is exact and the bf16 store rounds it like round_bf16 (plain drain and
    the split-K reductions)."""
    import torch
    from paper_2210_09603_b200 import Plan, ScheduleConfig
    _need_ref()
    L = W.ConvLayer("t", 64, 14, 256, 1, 1, 0, 1)
    d = W.conv_bn_dag(L, 2, residual=True)
    rng = port.Rng(610 + split_k)
    ins = {"X": rng.tensor((2, 64, 14, 14), True), "W": rng.tensor((256, 64, 1, 1), True),
           "Scale": rng.tensor((256,), True), "Shift": rng.tensor((256,), True),
           "R": rng.tensor((2, 256, 14, 14), True)}
    t = {k: dev(v, "bf16", "cl" if v.ndim == 4 else None) for k, v in ins.items()}
    z = torch.empty((2, 256, 14, 14), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    ex = Plan(d, ScheduleConfig(block_n=256, split_k=split_k)).bind([t[n] for n in d.inputs], [z])
    ex.launch()
    torch.cuda.synchronize()
    want = port.round_bf16(oracle_eval(d, ins, {"Z": (2, 256, 14, 14)})["Z"])
    assert np.array_equal(z.float().cpu().numpy(), want)
    assert ex.kernel_kind(0) == "gemm"
