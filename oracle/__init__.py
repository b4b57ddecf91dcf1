"""TEST INFRASTRUCTURE ONLY — the correctness oracle.  Never imported by the product.

Two layers, each pinned against the other by tests/test_oracle.py:

* ``oracle/_ref/libtaskmap_ref.so`` — the UNMODIFIED reference library
  (/root/reference/proj/src/*.cpp, compiled where it lies by oracle/Makefile)
  plus ``ref_shim.cpp``.  ``ref_eval`` is ``taskmap::reference_eval``
  (proj/src/compute_ir.cpp:418-466), the fp64/int64 element-by-element
  interpreter; it is the parity anchor for every kernel test.
* ``oracle.port`` — a numpy restatement of the reference's arithmetic for the
  five BASELINE configs (matmul+epilogue, batched matmul+scale, im2col conv +
  BN-fold + ReLU, FFN chain), each function citing the reference lines it
  restates.  It is the CPU "port" baseline and the fallback checker when the
  reference library cannot be rebuilt (it is pinned to the reference through
  the committed golden fixtures in tests/golden/).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Iterable, List, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libtaskmap_ref.so")

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is not None:
        return _ref
    if not ref_available():
        raise RuntimeError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
    L = ctypes.CDLL(REF_SO)
    P, I, U64, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
    CP = ctypes.c_char_p
    L.ref_eval.argtypes = [CP, I, ctypes.POINTER(CP), ctypes.POINTER(ctypes.POINTER(D)), I, ctypes.POINTER(CP),
                           ctypes.POINTER(ctypes.POINTER(D)), CP, I]
    L.ref_classify.argtypes = [CP, CP, ctypes.POINTER(I), CP, I]
    L.ref_validate.argtypes = [CP, CP, I]
    L.ref_mapping_info.argtypes = [CP, ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64),
                                   ctypes.POINTER(U64), CP, I]
    L.ref_mapping_assign.argtypes = [CP, U64, ctypes.POINTER(U64), U64, ctypes.POINTER(U64), CP, I]
    L.ref_mapping_text.argtypes = [CP, I, CP, I, CP, I]
    L.ref_mapping_compose_text.argtypes = [CP, CP, CP, I, CP, I]
    L.ref_rng_init.argtypes = [U64, ctypes.POINTER(U64)]
    L.ref_random.argtypes = [ctypes.POINTER(U64), I, I64, ctypes.POINTER(D)]
    L.ref_fold_bn.argtypes = [I64] + [ctypes.POINTER(D)] * 4 + [D, ctypes.POINTER(D), ctypes.POINTER(D)]
    L.ref_build.argtypes = [CP, ctypes.POINTER(I64), I, CP, I, CP, I]
    _ref = L
    return L


class RefError(RuntimeError):
    pass


def _err():
    return ctypes.create_string_buffer(4096)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def ref_eval(dag_json: str, inputs: Dict[str, np.ndarray], outputs: Sequence[str],
             shapes: Dict[str, Sequence[int]]) -> Dict[str, np.ndarray]:
    """taskmap::reference_eval on the DAG (inputs in logical row-major layout)."""
    L = ref_lib()
    names = list(inputs)
    arrs = [np.ascontiguousarray(inputs[n], dtype=np.float64) for n in names]
    outs = {o: np.zeros(int(np.prod(shapes[o])), dtype=np.float64) for o in outputs}
    in_names = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
    in_data = (ctypes.POINTER(ctypes.c_double) * len(names))(*[_dptr(a) for a in arrs])
    out_names = (ctypes.c_char_p * len(outputs))(*[o.encode() for o in outputs])
    out_data = (ctypes.POINTER(ctypes.c_double) * len(outputs))(*[_dptr(outs[o]) for o in outputs])
    e = _err()
    if L.ref_eval(dag_json.encode(), len(names), in_names, in_data, len(outputs), out_names, out_data, e, 4096):
        raise RefError(e.value.decode())
    return {o: outs[o].reshape(shapes[o]) for o in outputs}


def ref_classify(dag_json: str, node: str) -> int:
    L = ref_lib()
    out = ctypes.c_int()
    e = _err()
    if L.ref_classify(dag_json.encode(), node.encode(), ctypes.byref(out), e, 4096):
        raise RefError(e.value.decode())
    return out.value


def ref_validate(dag_json: str):
    e = _err()
    if ref_lib().ref_validate(dag_json.encode(), e, 4096):
        raise RefError(e.value.decode())


def ref_mapping_info(text: str):
    w, d, t = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    shape = (ctypes.c_uint64 * 16)()
    e = _err()
    if ref_lib().ref_mapping_info(text.encode(), ctypes.byref(w), ctypes.byref(d), ctypes.byref(t), shape, e, 4096):
        raise RefError(e.value.decode())
    return w.value, d.value, t.value, tuple(shape[i] for i in range(d.value))


def ref_mapping_assign(text: str, worker: int):
    _, dim, tpw, _ = ref_mapping_info(text)
    cap = max(1, dim * tpw)
    buf = (ctypes.c_uint64 * cap)()
    n = ctypes.c_uint64()
    e = _err()
    if ref_lib().ref_mapping_assign(text.encode(), int(worker), buf, cap, ctypes.byref(n), e, 4096):
        raise RefError(e.value.decode())
    return [tuple(buf[i * dim + k] for k in range(dim)) for i in range(n.value)]


def ref_mapping_text(text: str, visualize: bool = False) -> str:
    buf = ctypes.create_string_buffer(1 << 20)
    e = _err()
    if ref_lib().ref_mapping_text(text.encode(), int(visualize), buf, 1 << 20, e, 4096):
        raise RefError(e.value.decode())
    return buf.value.decode()


def ref_mapping_compose(a: str, b: str) -> str:
    buf = ctypes.create_string_buffer(1 << 16)
    e = _err()
    if ref_lib().ref_mapping_compose_text(a.encode(), b.encode(), buf, 1 << 16, e, 4096):
        raise RefError(e.value.decode())
    return buf.value.decode()


def ref_build(kind: str, args: Sequence[int]) -> str:
    arr = (ctypes.c_int64 * len(args))(*[int(a) for a in args])
    buf = ctypes.create_string_buffer(1 << 22)
    e = _err()
    if ref_lib().ref_build(kind.encode(), arr, len(args), buf, 1 << 22, e, 4096):
        raise RefError(e.value.decode())
    return buf.value.decode()


def ref_random_stream(seed: int, specs: Iterable[tuple]) -> List[np.ndarray]:
    """random_tensor draws from one Rng(seed) stream, in order; specs = (shape, is_int)."""
    L = ref_lib()
    st = ctypes.c_uint64()
    L.ref_rng_init(seed, ctypes.byref(st))
    out = []
    for shape, is_int in specs:
        n = int(np.prod(shape))
        a = np.zeros(n, dtype=np.float64)
        L.ref_random(ctypes.byref(st), int(is_int), n, _dptr(a))
        out.append(a.reshape(shape))
    return out


def ref_fold_bn(gamma, beta, mean, var, eps):
    c = len(gamma)
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (gamma, beta, mean, var)]
    scale = np.zeros(c)
    shift = np.zeros(c)
    ref_lib().ref_fold_bn(c, *[_dptr(a) for a in arrs], float(eps), _dptr(scale), _dptr(shift))
    return scale, shift
