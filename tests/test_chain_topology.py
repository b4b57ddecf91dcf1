"""The ResNet-50 chain's stage list (workloads.resnet50_stages, SURVEY.md §8 row
f2) and its DAGs, planned on the host: no GPU needed."""
from paper_2210_09603_b200 import Plan, ScheduleConfig
from paper_2210_09603_b200 import workloads as W


def test_stage_list_is_resnet50_v1_5():
    st = W.resnet50_stages()
    convs = [s for s in st if s.kind == "conv"]
    assert len(convs) == 53 and [s.kind for s in st[:2]] == ["conv", "maxpool"]
    assert [s.kind for s in st[-2:]] == ["avgpool", "linear"]
    table = {L.name: L for L in W.RESNET50}
    for s in convs:  # every conv has the shape of the sweep table's layer it reuses
        L = table[s.layer]
        assert (L.c, L.h, L.f, L.k, L.s, L.p) == (s.conv.c, s.conv.h, s.conv.f, s.conv.k, s.conv.s, s.conv.p)
    # per-table-layer use counts equal the table's `count` (53 layers, 24 shapes)
    for L in W.RESNET50:
        assert sum(s.layer == L.name for s in convs) == L.count, L.name
    # wiring: every stage reads activations produced earlier; residual adds only on c3
    seen = {"input"}
    for s in st:
        assert s.src in seen and (not s.res or s.res in seen), s
        assert bool(s.res) == s.dst.endswith(".c3")
        assert s.relu or s.dst.endswith(".ds")
        seen.add(s.dst)
    # v1.5: the stride sits on the 3x3 conv of each stage's first block
    assert [s.conv.s for s in convs if s.dst.endswith(".b0.c2")] == [1, 2, 2, 2]


def test_chain_dags_plan_to_the_expected_kernels():
    L = W.ConvLayer("t", 256, 14, 1024, 1, 1, 0, 1)
    kinds = lambda d: [k["kind"] for k in Plan(d, ScheduleConfig()).describe()["kernels"]]  # noqa: E731
    assert kinds(W.conv_bn_dag(L, 2, residual=True)) == ["gemm"]   # residual fused in the epilogue
    assert kinds(W.conv_bn_dag(L, 2, relu_out=False)) == ["gemm"]
    assert kinds(W.maxpool_dag(2, 64, 112)) == ["reduce"]
    assert kinds(W.avgpool_dag(2, 2048, 7)) == ["reduce"]
    assert kinds(W.linear_dag(32, 1000, 2048)) == ["gemm"]
