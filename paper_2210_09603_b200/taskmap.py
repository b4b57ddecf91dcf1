"""Python mirror of the taskmap API, bound to libtaskmap_b200.so through ctypes.

Names and argument meaning follow the reference headers:
  TaskMapping / parse_mapping      proj/include/taskmap/mapping.hpp:38-90
  expression builders              proj/include/taskmap/expr.hpp:40-70
  ComputeDAG / classify / builders proj/include/taskmap/compute_ir.hpp:25-114
and the spec-only scheduling API: ScheduleConfig,
schedule_space, partition, Plan (matmul_template + fuse_prologue/epilogue),
tune.  Errors raise TaskmapError (the reference's taskmap::Error).
"""
from __future__ import annotations

import ctypes
import enum
import json
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    return os.path.join(_HERE, "libtaskmap_b200.so")


class TaskmapError(RuntimeError):
    """taskmap::Error (proj/include/taskmap/common.hpp:10-12); .status is the C ABI code."""

    def __init__(self, msg: str, status: int = 2):
        super().__init__(msg)
        self.status = status


MAX_RANK = 8


class TmTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("shape", ctypes.c_int64 * MAX_RANK), ("stride", ctypes.c_int64 * MAX_RANK)]


class TmScheduleConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "block_m", "block_n", "block_k", "warp_m", "warp_n", "threads_per_block",
        "pipeline", "split_k", "stages", "raster", "grid", "math")]


_LIB = None


def load_library():
    """Loads the in-tree CUDA library; raises if it has not been built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise TaskmapError(f"{path} not found: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(path)
    P, I32, I64, U64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    sigs = {
        "tm_last_error": ([], ctypes.c_char_p),
        "tm_version": ([], ctypes.c_char_p),
        "tm_free": ([P], None),
        "tm_mapping_parse": ([ctypes.c_char_p, ctypes.POINTER(P)], I32),
        "tm_mapping_free": ([P], None),
        "tm_mapping_info": ([P, ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64)], I32),
        "tm_mapping_assign": ([P, U64, ctypes.POINTER(U64), SZ, ctypes.POINTER(SZ)], I32),
        "tm_mapping_lowered_assign": ([P, U64, ctypes.POINTER(U64), SZ, ctypes.POINTER(SZ)], I32),
        "tm_mapping_text": ([P, ctypes.c_int, ctypes.POINTER(P)], I32),
        "tm_kernel_mapping_assign": ([I32, U64, ctypes.POINTER(U64), SZ, ctypes.POINTER(SZ)], I32),
        "tm_classify": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(I32)], I32),
        "tm_partition": ([ctypes.c_char_p, ctypes.POINTER(P)], I32),
        "tm_build_dag": ([ctypes.c_char_p, ctypes.POINTER(I64), I32, ctypes.POINTER(P)], I32),
        "tm_schedule_space": ([ctypes.c_char_p, ctypes.POINTER(TmScheduleConfig), I32, ctypes.POINTER(I32)], I32),
        "tm_plan_create": ([ctypes.c_char_p, ctypes.POINTER(TmScheduleConfig), I32, ctypes.POINTER(P)], I32),
        "tm_plan_destroy": ([P], None),
        "tm_plan_describe": ([P, ctypes.POINTER(P)], I32),
        "tm_exec_create": ([P, ctypes.POINTER(TmTensor), I32, ctypes.POINTER(TmTensor), I32, ctypes.POINTER(P)], I32),
        "tm_exec_destroy": ([P], None),
        "tm_exec_launch": ([P, P], I32),
        "tm_exec_num_launches": ([P], I32),
        "tm_exec_kernel_info": ([P, I32] + [ctypes.POINTER(I32)] * 6, I32),
        "tm_exec_kernel_kind": ([P, I32, ctypes.POINTER(I32)], I32),
        "tm_exec_trace": ([P, I32, ctypes.POINTER(I64), SZ], I32),
        "tm_plan_launch": ([P, ctypes.POINTER(TmTensor), I32, ctypes.POINTER(TmTensor), I32, P], I32),
        "tm_graph_create": ([ctypes.POINTER(P), I32, I32, ctypes.POINTER(P)], I32),
        "tm_graph_launch": ([P, P], I32),
        "tm_graph_exec_ms": ([P, ctypes.POINTER(ctypes.c_float), I32], I32),
        "tm_graph_destroy": ([P], None),
        "tm_tune": ([ctypes.c_char_p, ctypes.POINTER(TmTensor), I32, ctypes.POINTER(TmTensor), I32, I32, I32,
                     ctypes.POINTER(TmScheduleConfig), ctypes.POINTER(P)], I32),
        "tm_dag_eval": ([ctypes.c_char_p, ctypes.POINTER(TmTensor), I32, ctypes.POINTER(TmTensor), I32, I32, P], I32),
    }
    for name, (args, res) in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _LIB = L
    return L


def _check(status: int):
    if status != 0:
        msg = load_library().tm_last_error().decode()
        raise TaskmapError(msg, status)


def _take_string(p: ctypes.c_void_p) -> str:
    s = ctypes.cast(p, ctypes.c_char_p).value.decode()
    load_library().tm_free(p)
    return s


# ---------------------------------------------------------------- enums --
class DType(enum.Enum):
    F32 = "f32"
    I32 = "i32"


class BinOp(enum.Enum):
    Add = "add"; Sub = "sub"; Mul = "mul"; Div = "div"; Mod = "mod"; Min = "min"; Max = "max"
    And = "and"; Or = "or"; Lt = "lt"; Le = "le"; Gt = "gt"; Ge = "ge"; Eq = "eq"; Ne = "ne"


class UnOp(enum.Enum):
    Neg = "neg"; Relu = "relu"; Exp = "exp"; Sqrt = "sqrt"; CastF32 = "f32"; CastI32 = "i32"


class Combiner(enum.Enum):
    Sum = "sum"; Max = "max"; Min = "min"


class OpClass(enum.IntEnum):
    Reduction = 0
    Injective = 1
    Bijective = 2


# -------------------------------------------------------- task mappings --
class TaskMapping:
    """An immutable task mapping value (mapping.hpp:38-83), backed by the C++ object."""

    def __init__(self, text: str):
        L = load_library()
        h = ctypes.c_void_p()
        _check(L.tm_mapping_parse(text.encode(), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.tm_mapping_free(self._h)
            self._h = None

    @staticmethod
    def repeat(*dims) -> "TaskMapping":
        return TaskMapping("repeat(" + ", ".join(str(int(d)) for d in dims) + ")")

    @staticmethod
    def spatial(*dims) -> "TaskMapping":
        return TaskMapping("spatial(" + ", ".join(str(int(d)) for d in dims) + ")")

    def __mul__(self, other: "TaskMapping") -> "TaskMapping":
        return TaskMapping(f"({self.to_text()}) * ({other.to_text()})")

    def _info(self):
        nw, dim, tpw = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        shape = (ctypes.c_uint64 * 16)()
        _check(load_library().tm_mapping_info(self._h, ctypes.byref(nw), ctypes.byref(dim), ctypes.byref(tpw), shape))
        return nw.value, dim.value, tpw.value, tuple(shape[i] for i in range(dim.value))

    @property
    def num_workers(self) -> int:
        return self._info()[0]

    @property
    def task_dim(self) -> int:
        return self._info()[1]

    @property
    def tasks_per_worker(self) -> int:
        return self._info()[2]

    @property
    def task_shape(self):
        return self._info()[3]

    def _assign(self, fn, worker):
        _, dim, tpw, _ = self._info()
        cap = max(1, tpw * dim)
        buf = (ctypes.c_uint64 * cap)()
        n = ctypes.c_size_t()
        _check(fn(self._h, int(worker), buf, cap, ctypes.byref(n)))
        return [tuple(buf[i * dim + d] for d in range(dim)) for i in range(n.value)]

    def assign(self, worker: int):
        return self._assign(load_library().tm_mapping_assign, worker)

    def lowered_assign(self, worker: int):
        """Closed-form device lowering (DevMapping) evaluated on the host."""
        return self._assign(load_library().tm_mapping_lowered_assign, worker)

    def to_text(self) -> str:
        p = ctypes.c_void_p()
        _check(load_library().tm_mapping_text(self._h, 0, ctypes.byref(p)))
        return _take_string(p)

    def visualize(self) -> str:
        p = ctypes.c_void_p()
        _check(load_library().tm_mapping_text(self._h, 1, ctypes.byref(p)))
        return _take_string(p)

    def __repr__(self):
        return f"TaskMapping({self.to_text()!r})"


def parse_mapping(text: str) -> TaskMapping:
    return TaskMapping(text)


# ---------------------------------------------------------- expressions --
# Expressions are the JSON wire form (prefix lists) understood by the C++ side.
def imm(v: int):
    return ["i", int(v)]


def fimm(v: float):
    return ["f", float(v)]


def var(name: str):
    return ["v", name]


def load(buffer: str, indices: Sequence):
    return ["load", buffer, *indices]


def select(c, t, e):
    return ["select", c, t, e]


def binary(op: BinOp, a, b):
    if op in (BinOp.Div, BinOp.Mod) and b == ["i", 0]:
        raise TaskmapError("division/modulo by zero constant")
    return [op.value, a, b]


def unary(op: UnOp, a):
    return [op.value, a]


def add(a, b): return binary(BinOp.Add, a, b)
def sub(a, b): return binary(BinOp.Sub, a, b)
def mul(a, b): return binary(BinOp.Mul, a, b)
def div(a, b): return binary(BinOp.Div, a, b)
def mod(a, b): return binary(BinOp.Mod, a, b)
def minimum(a, b): return binary(BinOp.Min, a, b)
def maximum(a, b): return binary(BinOp.Max, a, b)
def land(a, b): return binary(BinOp.And, a, b)
def lor(a, b): return binary(BinOp.Or, a, b)
def lt(a, b): return binary(BinOp.Lt, a, b)
def le(a, b): return binary(BinOp.Le, a, b)
def gt(a, b): return binary(BinOp.Gt, a, b)
def ge(a, b): return binary(BinOp.Ge, a, b)
def eq(a, b): return binary(BinOp.Eq, a, b)
def ne(a, b): return binary(BinOp.Ne, a, b)
def neg(a): return unary(UnOp.Neg, a)
def relu(a): return unary(UnOp.Relu, a)
def exp(a): return unary(UnOp.Exp, a)
def sqrt(a): return unary(UnOp.Sqrt, a)


def zero_of(dt: DType):
    return fimm(0.0) if dt == DType.F32 else imm(0)


def gelu_tanh(x):
    """tanh-form GELU written with Exp/Div (the IR has no tanh, expr.hpp:16); same tree as taskmap::gelu_tanh."""
    x3 = mul(mul(x, x), x)
    inner = mul(fimm(0.7978845608028654), add(x, mul(fimm(0.044715), x3)))
    t = sub(fimm(1.0), div(fimm(2.0), add(exp(mul(fimm(2.0), inner)), fimm(1.0))))
    return mul(mul(fimm(0.5), x), add(fimm(1.0), t))


# ------------------------------------------------------------------ DAG --
@dataclass
class Axis:
    name: str
    extent: int


@dataclass
class TensorNode:
    name: str
    shape: List[int]
    dtype: DType = DType.F32
    kind: str = "input"                  # input | compute | reduce
    axes: List[Axis] = field(default_factory=list)
    reduce_axes: List[Axis] = field(default_factory=list)
    combiner: Combiner = Combiner.Sum
    value: Optional[list] = None

    def to_obj(self):
        o = {"name": self.name, "shape": list(self.shape), "dtype": self.dtype.value, "kind": self.kind}
        if self.kind != "input":
            o["axes"] = [[a.name, a.extent] for a in self.axes]
            o["value"] = self.value
            if self.kind == "reduce":
                o["reduce_axes"] = [[a.name, a.extent] for a in self.reduce_axes]
                o["combiner"] = self.combiner.value
        return o

    @staticmethod
    def from_obj(o) -> "TensorNode":
        n = TensorNode(o["name"], list(o["shape"]), DType(o.get("dtype", "f32")), o.get("kind", "input"))
        if n.kind != "input":
            n.axes = [Axis(a[0], a[1]) for a in o.get("axes", [])]
            n.reduce_axes = [Axis(a[0], a[1]) for a in o.get("reduce_axes", [])]
            n.combiner = Combiner(o.get("combiner", "sum"))
            n.value = o["value"]
        return n


def compute(name: str, axes: Sequence[Axis], value, dtype: DType = DType.F32) -> TensorNode:
    return TensorNode(name, [a.extent for a in axes], dtype, "compute", list(axes), [], Combiner.Sum, value)


@dataclass
class ComputeDAG:
    nodes: List[TensorNode] = field(default_factory=list)
    inputs: List[str] = field(default_factory=list)
    outputs: List[str] = field(default_factory=list)

    def find(self, name: str) -> Optional[TensorNode]:
        return next((n for n in self.nodes if n.name == name), None)

    def at(self, name: str) -> TensorNode:
        n = self.find(name)
        if n is None:
            raise TaskmapError(f"no tensor named '{name}' in DAG")
        return n

    def to_json(self) -> str:
        return json.dumps({"nodes": [n.to_obj() for n in self.nodes], "inputs": self.inputs, "outputs": self.outputs})

    @staticmethod
    def from_json(text: str) -> "ComputeDAG":
        o = json.loads(text)
        return ComputeDAG([TensorNode.from_obj(n) for n in o["nodes"]], list(o["inputs"]), list(o["outputs"]))

    def add_input(self, name: str, shape, dtype: DType = DType.F32):
        self.nodes.append(TensorNode(name, list(shape), dtype))
        self.inputs.append(name)
        return self

    def add_compute(self, name: str, axes, value, dtype: DType = DType.F32):
        self.nodes.append(compute(name, [a if isinstance(a, Axis) else Axis(*a) for a in axes], value, dtype))
        return self

    def validate(self):
        classify(self, self.nodes[-1].name) if any(n.kind != "input" for n in self.nodes) else None


def classify(dag: ComputeDAG, node: str) -> OpClass:
    out = ctypes.c_int32()
    _check(load_library().tm_classify(dag.to_json().encode(), node.encode(), ctypes.byref(out)))
    return OpClass(out.value)


def partition(dag: ComputeDAG):
    p = ctypes.c_void_p()
    _check(load_library().tm_partition(dag.to_json().encode(), ctypes.byref(p)))
    return json.loads(_take_string(p))


def _build(kind: str, args: Sequence[int]) -> ComputeDAG:
    arr = (ctypes.c_int64 * len(args))(*[int(a) for a in args])
    p = ctypes.c_void_p()
    _check(load_library().tm_build_dag(kind.encode(), arr, len(args), ctypes.byref(p)))
    return ComputeDAG.from_json(_take_string(p))


def _dt(dtype: DType) -> int:
    return 0 if dtype == DType.F32 else 1


def matmul_dag(m, n, k, dtype: DType = DType.F32) -> ComputeDAG:
    return _build("matmul", [m, n, k, _dt(dtype)])


def conv2d_im2col_dag(n, c, h, w, f, kh, kw, stride, pad, dtype: DType = DType.F32) -> ComputeDAG:
    return _build("conv2d_im2col", [n, c, h, w, f, kh, kw, stride, pad, _dt(dtype)])


def batchnorm_inference_dag(n, c, h, w, dtype: DType = DType.F32) -> ComputeDAG:
    return _build("batchnorm", [n, c, h, w, _dt(dtype)])


def transpose_dag(shape, perm, dtype: DType = DType.F32) -> ComputeDAG:
    return _build("transpose", [_dt(dtype), len(shape), *shape, *perm])


def reshape_dag(in_shape, out_shape, dtype: DType = DType.F32) -> ComputeDAG:
    return _build("reshape", [_dt(dtype), len(in_shape), *in_shape, len(out_shape), *out_shape])


# ----------------------------------------------------------- scheduling --
_MATH = {"auto": 0, "bf16": 1, "tf32": 2, "fp32_simt": 3, "halo": 4}


@dataclass
class ScheduleConfig:
    """SPEC.md:276-279 fields + the Blackwell fields (see include/taskmap/schedule.hpp)."""
    block_m: int = 128
    block_n: int = 128
    block_k: int = 64
    warp_m: int = 4
    warp_n: int = 1
    threads_per_block: int = 288
    pipeline: bool = True
    split_k: int = 1
    stages: int = 0
    raster: int = 0
    grid: int = 0
    math: str = "auto"

    def to_c(self) -> TmScheduleConfig:
        c = TmScheduleConfig()
        for f in ("block_m", "block_n", "block_k", "warp_m", "warp_n", "threads_per_block", "split_k",
                  "stages", "raster", "grid"):
            setattr(c, f, int(getattr(self, f)))
        c.pipeline = int(bool(self.pipeline))
        c.math = _MATH[self.math]
        return c

    @staticmethod
    def from_c(c: TmScheduleConfig) -> "ScheduleConfig":
        inv = {v: k for k, v in _MATH.items()}
        return ScheduleConfig(c.block_m, c.block_n, c.block_k, c.warp_m, c.warp_n, c.threads_per_block,
                              bool(c.pipeline), c.split_k, c.stages, c.raster, c.grid, inv.get(c.math, "auto"))


def schedule_space(op_kind: str = "matmul") -> List[ScheduleConfig]:
    n = ctypes.c_int32()
    _check(load_library().tm_schedule_space(op_kind.encode(), None, 0, ctypes.byref(n)))
    buf = (TmScheduleConfig * n.value)()
    _check(load_library().tm_schedule_space(op_kind.encode(), buf, n.value, ctypes.byref(n)))
    return [ScheduleConfig.from_c(buf[i]) for i in range(n.value)]


# ------------------------------------------------------------ execution --
_TORCH_DT = None


def _tensor_arg(t) -> TmTensor:
    """torch.Tensor (device memory, any strides) -> tm_tensor."""
    import torch
    global _TORCH_DT
    if _TORCH_DT is None:
        _TORCH_DT = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
    if t.dtype not in _TORCH_DT:
        raise TaskmapError(f"unsupported tensor dtype {t.dtype}")
    a = TmTensor()
    a.data = t.data_ptr()
    a.dtype = _TORCH_DT[t.dtype]
    a.rank = t.dim()
    for d in range(t.dim()):
        a.shape[d] = t.shape[d]
        a.stride[d] = t.stride(d)
    return a


class Exec:
    """A plan bound to concrete device tensors (tm_exec)."""

    def __init__(self, plan: "Plan", inputs, outputs):
        self._keep = (list(inputs), list(outputs))
        ins = (TmTensor * max(1, len(inputs)))(*[_tensor_arg(t) for t in inputs])
        outs = (TmTensor * max(1, len(outputs)))(*[_tensor_arg(t) for t in outputs])
        h = ctypes.c_void_p()
        _check(load_library().tm_exec_create(plan._h, ins, len(inputs), outs, len(outputs), ctypes.byref(h)))
        self._h = h

    @property
    def num_launches(self) -> int:
        return load_library().tm_exec_num_launches(self._h)

    def kernel_info(self, index: int = 0) -> dict:
        v = [ctypes.c_int32() for _ in range(6)]
        _check(load_library().tm_exec_kernel_info(self._h, index, *[ctypes.byref(x) for x in v]))
        return dict(zip(("grid", "cta_group", "block_n", "split_k", "a_loader", "b_loader"), [x.value for x in v]))

    KERNEL_KINDS = ("gemm", "simt", "rowband", "halo", "rule-interp", "rule-generated")

    def kernel_kind(self, index: int = 0) -> str:
        """Kernel family of launch `index` (tm_exec_kernel_kind)."""
        k = ctypes.c_int32()
        _check(load_library().tm_exec_kernel_kind(self._h, index, ctypes.byref(k)))
        return self.KERNEL_KINDS[k.value]

    def trace(self, index: int = 0):
        """Per-tile role timeline (needs TMB_TRACE=1 at bind time): int64 [grid, 64, 8]."""
        import numpy as np
        g = self.kernel_info(index)["grid"]
        buf = np.zeros((g, 64, 16), dtype=np.int64)
        _check(load_library().tm_exec_trace(self._h, index, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                            buf.size))
        return buf

    def launch(self, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(load_library().tm_exec_launch(self._h, ctypes.c_void_p(s.cuda_stream)))

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.tm_exec_destroy(self._h)
            self._h = None


class Graph:
    """A CUDA graph replaying a sequence of bound execs with one launch (tm_graph).

    timed=True records an event around every exec; exec_ms() then returns the
    per-exec device time (ms) of the most recent launch (after a synchronize)."""

    def __init__(self, execs, timed: bool = False):
        self._execs = list(execs)  # the graph references their buffers
        arr = (ctypes.c_void_p * max(1, len(self._execs)))(*[e._h.value for e in self._execs])
        h = ctypes.c_void_p()
        _check(load_library().tm_graph_create(arr, len(self._execs), int(timed), ctypes.byref(h)))
        self._h = h

    def launch(self, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(load_library().tm_graph_launch(self._h, ctypes.c_void_p(s.cuda_stream)))

    def exec_ms(self):
        n = len(self._execs)
        buf = (ctypes.c_float * max(1, n))()
        _check(load_library().tm_graph_exec_ms(self._h, buf, n))
        return [buf[i] for i in range(n)]

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.tm_graph_destroy(self._h)
            self._h = None


class Plan:
    """partition + fuse + schedule a DAG onto the sm_100a tensor programs (tm_plan)."""

    def __init__(self, dag: ComputeDAG, config: Optional[ScheduleConfig] = None, device: Optional[int] = None):
        self.dag = dag
        self.config = config or ScheduleConfig()
        device = _resolve_device(device)
        c = self.config.to_c()
        h = ctypes.c_void_p()
        _check(load_library().tm_plan_create(dag.to_json().encode(), ctypes.byref(c), int(device), ctypes.byref(h)))
        self._h = h

    def describe(self):
        p = ctypes.c_void_p()
        _check(load_library().tm_plan_describe(self._h, ctypes.byref(p)))
        return json.loads(_take_string(p))

    def bind(self, inputs, outputs) -> Exec:
        return Exec(self, inputs, outputs)

    def __call__(self, inputs, outputs, stream=None):
        e = self.bind(inputs, outputs)
        e.launch(stream)
        return e

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.tm_plan_destroy(self._h)
            self._h = None


def _resolve_device(device: Optional[int], tensors=()) -> int:
    """The CUDA device a plan binds / tunes on: explicit, else that of the first
    CUDA tensor given, else torch's current device (one process per GPU: rank r
    must not fall back to device 0)."""
    if device is not None:
        return int(device)
    for t in tensors:
        if getattr(t, "is_cuda", False):
            return int(t.device.index)
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except Exception:  # noqa: BLE001
        pass
    return 0


def tune(dag: ComputeDAG, inputs, outputs, device: Optional[int] = None, reps: int = 5):
    """Exhaustive on-device tuning over schedule_space; returns (best, report).

    Every config is verified against the device DAG interpreter on two seeded
    inputs before it is timed; an incorrect config aborts tuning with a
    TaskmapError of status 1 (TM_ERR_CORRECTNESS) whose .report holds the
    TuneReport."""
    device = _resolve_device(device, list(inputs) + list(outputs))
    ins = (TmTensor * max(1, len(inputs)))(*[_tensor_arg(t) for t in inputs])
    outs = (TmTensor * max(1, len(outputs)))(*[_tensor_arg(t) for t in outputs])
    best = TmScheduleConfig()
    p = ctypes.c_void_p()
    L = load_library()
    status = L.tm_tune(dag.to_json().encode(), ins, len(inputs), outs, len(outputs), int(device),
                       int(reps), ctypes.byref(best), ctypes.byref(p))
    report = json.loads(_take_string(p)) if p.value else None
    if status != 0:
        err = TaskmapError(L.tm_last_error().decode(), status)
        err.report = report
        raise err
    return ScheduleConfig.from_c(best), report


def dag_eval(dag: ComputeDAG, inputs, outputs, device: Optional[int] = None, stream=None):
    """The reference interpreter's semantics re-run on the device (tm_dag_eval): writes dag.outputs into `outputs`."""
    import torch
    device = _resolve_device(device, list(inputs) + list(outputs))
    ins = (TmTensor * max(1, len(inputs)))(*[_tensor_arg(t) for t in inputs])
    outs = (TmTensor * max(1, len(outputs)))(*[_tensor_arg(t) for t in outputs])
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(load_library().tm_dag_eval(dag.to_json().encode(), ins, len(inputs), outs, len(outputs), int(device),
                                      ctypes.c_void_p(s.cuda_stream)))
