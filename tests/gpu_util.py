"""Helpers for GPU parity tests: upload oracle inputs, run a Plan, fetch results."""
import numpy as np

import oracle
from oracle import port
from paper_2210_09603_b200 import Plan, ScheduleConfig


def torch():
    import torch as _t
    return _t


def dev(a, dtype="bf16", layout=None):
    """float64 numpy -> CUDA tensor of dtype; layout 'cl' = channels-last strides for 4-D,
    't' = transposed storage (same logical values, column-major strides) for 2-D/3-D."""
    t = torch()
    tdt = {"bf16": t.bfloat16, "f32": t.float32, "f16": t.float16}[dtype]
    x = t.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(tdt)
    if layout == "cl":
        x = x.contiguous(memory_format=t.channels_last)
    elif layout == "cl8":
        # NCHW logical view over a 16-byte padded channels-last buffer [N, H, W, 8];
        # the pad channels hold NaN to prove they are never read (TMA zero-fills them)
        n, c, h, w = x.shape
        buf = t.full((n, h, w, 8), float("nan"), dtype=tdt)
        buf[..., :c] = x.permute(0, 2, 3, 1)
        buf = buf.cuda()
        return buf.as_strided((n, c, h, w), (h * w * 8, 1, w * 8, 8))
    elif layout == "t":
        x = x.transpose(-1, -2).contiguous().transpose(-1, -2)
    return x.cuda()


def rounded(a, dtype):
    if dtype == "bf16":
        return port.round_bf16(a)
    if dtype == "tf32":
        return port.round_tf32(a)
    return np.asarray(a, np.float32).astype(np.float64)


def run(dag, inputs, out_shapes, out_dtype="f32", cfg=None):
    """inputs: dict name -> CUDA tensor (ordered as dag.inputs). Returns dict name -> float64 numpy."""
    t = torch()
    tdt = {"bf16": t.bfloat16, "f32": t.float32, "f16": t.float16}[out_dtype]
    outs = {o: t.full(tuple(out_shapes[o]), float("nan"), dtype=tdt, device="cuda") for o in dag.outputs}
    plan = Plan(dag, cfg or ScheduleConfig())
    ex = plan.bind([inputs[n] for n in dag.inputs], [outs[o] for o in dag.outputs])
    ex.launch()
    t.cuda.synchronize()
    return {o: outs[o].float().cpu().numpy().astype(np.float64) for o in dag.outputs}, plan


def oracle_eval(dag, inputs_np, out_shapes):
    """reference_eval (the real reference library) on the DAG."""
    return oracle.ref_eval(dag.to_json(), inputs_np, list(out_shapes), out_shapes)


def have_ref():
    return oracle.ref_available()
