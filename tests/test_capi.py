"""The C-ABI library loads, exports exactly the entry points include/taskmap_b200.h
declares, and maps errors to the spec's status codes (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2210_09603_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "taskmap_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tm_[a-z_]+)\s*\(", text)))


def test_header_symbols_all_exported():
    lib = ctypes.CDLL(pkg.lib_path())
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in taskmap_b200.h but not exported"


def test_only_declared_symbols_exported():
    """The library exports exactly the C ABI of include/taskmap_b200.h (extern "C" tm_*)
    plus the C++ boundary in namespace taskmap (include/taskmap/*.hpp); nothing else."""
    out = subprocess.run(["nm", "-D", "--defined-only", pkg.lib_path()], capture_output=True, text=True).stdout
    syms = [l.split()[-1] for l in out.splitlines() if " T " in l or " W " in l]
    c_syms = [s for s in syms if s.startswith("tm_")]
    assert sorted(c_syms) == declared()
    cxx = subprocess.run(["c++filt"], input="\n".join(s for s in syms if not s.startswith("tm_")),
                         capture_output=True, text=True).stdout.split("\n")
    cxx = [c for c in cxx if c]
    assert cxx and all(c.startswith("taskmap::") or "taskmap::" in c.split("(")[0] for c in cxx), cxx[:5]


def test_status_codes_and_last_error():
    lib = pkg.load_library()
    h = ctypes.c_void_p()
    assert lib.tm_mapping_parse(b"repeat(2", ctypes.byref(h)) == 2        # TM_ERR_USAGE
    assert b"parse error" in lib.tm_last_error()
    cls = ctypes.c_int32()
    assert lib.tm_classify(b"{not json", b"Y", ctypes.byref(cls)) == 2
    assert b"json" in lib.tm_last_error()
    assert lib.tm_mapping_parse(b"spatial(2, 2)", ctypes.byref(h)) == 0
    assert lib.tm_last_error() == b""
    lib.tm_mapping_free(h)
    assert b"sm_100a" in lib.tm_version()


def test_unsupported_status_code():
    from paper_2210_09603_b200 import Axis, ComputeDAG, TensorNode, load, var, Plan, TaskmapError
    from paper_2210_09603_b200.taskmap import Combiner
    d = ComputeDAG()
    d.add_input("X", [1] * 9)
    ax = [Axis(f"a{i}", 1) for i in range(9)]
    d.nodes.append(TensorNode("Y", [1] * 9, kind="compute", axes=ax, value=load("X", [var(a.name) for a in ax])))
    d.outputs = ["Y"]
    with pytest.raises(TaskmapError) as e:
        Plan(d)
    assert e.value.status == 4  # TM_ERR_UNSUPPORTED: a valid 9-d DAG beyond the rule kernel's 8 axes


def test_product_never_imports_oracle():
    """The shipped package must not route through the oracle (CPU fallback ban)."""
    pkgdir = os.path.join(ROOT, "paper_2210_09603_b200")
    for dirpath, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h", ".hpp")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "reference_eval" not in src or f.endswith((".cpp", ".cuh", ".h", ".hpp", ".cu")), f
    out = subprocess.run(["nm", "-D", pkg.lib_path()], capture_output=True, text=True).stdout
    assert "ref_eval" not in out and "reference_eval" not in out
