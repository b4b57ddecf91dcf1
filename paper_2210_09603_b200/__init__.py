"""paper_2210_09603_b200 — B200-native task-mapping tensor programs (Hidet, arXiv 2210.09603).

Python mirror of the reference's C++ operator / task-mapping API
(/root/reference/proj/include/taskmap/*.hpp) over the C ABI in
include/taskmap_b200.h.  The compute path is the in-tree CUDA library
libtaskmap_b200.so (sm_100a); importing this package never falls back to a
CPU implementation — if the library is missing, every entry point raises.
"""
from .taskmap import (  # noqa: F401
    BinOp, UnOp, DType, Combiner, OpClass, TaskMapping, parse_mapping,
    imm, fimm, var, load, select, binary, unary, add, sub, mul, div, mod, minimum, maximum,
    land, lor, lt, le, gt, ge, eq, ne, neg, relu, exp, sqrt, gelu_tanh, zero_of,
    Axis, TensorNode, ComputeDAG, classify, partition,
    matmul_dag, conv2d_im2col_dag, batchnorm_inference_dag, transpose_dag, reshape_dag,
    ScheduleConfig, schedule_space, Plan, Exec, Graph, tune, dag_eval, TaskmapError, lib_path, load_library,
)

__all__ = [n for n in dir() if not n.startswith("_")]
