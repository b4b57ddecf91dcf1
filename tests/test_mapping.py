"""Task-mapping algebra parity with the reference (mapping.cpp) — CPU only.

Golden answers come from the reference library (tests/golden, made by
make_golden.py); SPEC.md acceptance criteria 1-3 (associativity, Fig. 5
composition, coverage bijection) are checked on the product's TaskMapping, and
the closed-form device lowering (DevMapping, used by the kernels' CTA->tile
scheduler) must equal assign() bit for bit.
"""
import itertools
import json
import os
import random

import pytest

import oracle
from paper_2210_09603_b200 import TaskMapping, TaskmapError, parse_mapping

HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))


@pytest.mark.parametrize("m", META["mappings"], ids=[m["text"][:40] for m in META["mappings"]])
def test_mapping_matches_reference_golden(m):
    tm = TaskMapping(m["text"])
    assert tm.num_workers == m["workers"]
    assert tm.task_dim == m["task_dim"]
    assert tm.tasks_per_worker == m["tasks_per_worker"]
    assert list(tm.task_shape) == m["shape"]
    assert tm.to_text() == m["canonical"]
    if m["visualize"] is not None:
        assert tm.visualize() == m["visualize"]
    for w, tasks in zip(m["workers_checked"], m["assign"]):
        assert [list(t) for t in tm.assign(w)] == [list(t) for t in tasks]
        if "custom" not in m["text"]:
            assert [list(t) for t in tm.lowered_assign(w)] == [list(t) for t in tasks]


def test_fig5_cooperative_load():
    """SPEC.md:75 / :525: repeat(4,1)*spatial(16,8): 128 workers, 64x8, w0 = rows 0,16,32,48."""
    m = TaskMapping.repeat(4, 1) * TaskMapping.spatial(16, 8)
    assert m.num_workers == 128 and m.task_shape == (64, 8)
    assert m.assign(0) == [(0, 0), (16, 0), (32, 0), (48, 0)]
    assert m.assign(9) == [(1, 1), (17, 1), (33, 1), (49, 1)]


def test_paper_cuda_core_mapping():
    """spatial(4,2)*repeat(2,2)*spatial(4,8)*repeat(4,4): 256 workers, 128x128."""
    m = parse_mapping("spatial(4, 2) * repeat(2, 2) * spatial(4, 8) * repeat(4, 4)")
    assert m.num_workers == 256 and m.task_shape == (128, 128) and m.tasks_per_worker == 64
    assert m.assign(0)[:4] == [(0, 0), (0, 1), (0, 2), (0, 3)]
    assert m.assign(32)[:2] == [(0, 64), (0, 65)]


def test_errors_match_reference_messages():
    with pytest.raises(TaskmapError, match="cannot compose mappings with task dimensions 1 and 2"):
        TaskMapping("repeat(2) * spatial(2, 2)")
    with pytest.raises(TaskmapError, match="worker id 4 out of range for 4 workers"):
        TaskMapping.spatial(2, 2).assign(4)
    with pytest.raises(TaskmapError, match="task shape extents must be positive"):
        TaskMapping("repeat(0)")
    with pytest.raises(TaskmapError, match="parse error"):
        TaskMapping("repeat(2")
    if oracle.ref_available():
        with pytest.raises(oracle.RefError, match="cannot compose mappings with task dimensions 1 and 2"):
            oracle.ref_mapping_compose("repeat(2)", "spatial(2, 2)")


def _random_chain(rng, dim, natoms):
    return " * ".join(f"{rng.choice(['repeat', 'spatial'])}({', '.join(str(rng.randint(1, 4)) for _ in range(dim))})"
                      for _ in range(natoms))


def test_associativity_500_triples():
    """SPEC.md acceptance 1: (f1*f2)*f3 == f1*(f2*f3) on every worker."""
    rng = random.Random(11)
    for _ in range(500):
        dim = rng.randint(1, 3)
        a, b, c = (_random_chain(rng, dim, 1) for _ in range(3))
        left, right = TaskMapping(f"({a} * {b}) * {c}"), TaskMapping(f"{a} * ({b} * {c})")
        assert left.num_workers == right.num_workers
        for w in range(left.num_workers):
            assert left.assign(w) == right.assign(w)


def test_coverage_bijection_200_compositions():
    """SPEC.md acceptance 3: every task of the domain appears exactly once."""
    rng = random.Random(13)
    for _ in range(200):
        dim = rng.randint(1, 3)
        m = TaskMapping(_random_chain(rng, dim, rng.randint(1, 4)))
        seen = [t for w in range(m.num_workers) for t in m.assign(w)]
        assert len(seen) == len(set(seen))
        assert set(seen) == set(itertools.product(*[range(d) for d in m.task_shape]))


@pytest.mark.parametrize("which,text", [
    (0, "spatial(4, 2) * repeat(2, 2) * spatial(4, 8) * repeat(4, 4)"),
    (1, "repeat(4, 1) * spatial(32, 8)"),
    (2, "repeat(1, 4) * spatial(8, 32)")])
def test_kernel_compiled_mappings_equal_reference_assign(which, text):
    """The compile-time (constexpr) mappings inside the fp32 CUDA-core kernel produce
    exactly the task lists of the reference's assign() for the same mapping text."""
    import ctypes
    from paper_2210_09603_b200.taskmap import load_library
    lib = load_library()
    ref = oracle.ref_mapping_assign if oracle.ref_available() else (lambda t, w: TaskMapping(t).assign(w))
    for w in range(256):
        buf = (ctypes.c_uint64 * 4096)()
        n = ctypes.c_size_t()
        assert lib.tm_kernel_mapping_assign(which, w, buf, 4096, ctypes.byref(n)) == 0
        got = [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]
        assert got == [tuple(t) for t in ref(text, w)]


def test_lowering_equals_assign_random_chains():
    """the closed-form per-worker index (device DevMapping) equals assign()."""
    rng = random.Random(17)
    for _ in range(300):
        dim = rng.randint(1, 3)
        m = TaskMapping(_random_chain(rng, dim, rng.randint(1, 6)))
        for w in range(m.num_workers):
            assert m.lowered_assign(w) == m.assign(w)
