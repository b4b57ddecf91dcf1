#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) on the kernels added late in
# round 2: the NVRTC-generated rule / reduce kernels (elem, tree, lane-group,
# split-CTA with its atomic ticket) and the residual-before-ReLU compact drain of
# the network chain (plain and split-K).
OUT=gpurun_out/san_r02b
mkdir -p $OUT
cat > $OUT/cases.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from gpu_util import dev, run, oracle_eval
from oracle import port
from paper_2210_09603_b200 import ScheduleConfig, workloads as W
case = sys.argv[1]
if case in ("gen_softmax", "interp_softmax"):
    if case.startswith("interp"):
        os.environ["TMB_RULE_INTERP"] = "1"
    import test_gpu_rule as T
    d = T._softmax_dag(64, 300)
    x = port.Rng(904).tensor((64, 300))
    got, _ = run(d, {"X": dev(x, "f32")}, {"P": (64, 300)})
    ok = port.max_rel_error(got["P"], oracle_eval(d, {"X": x}, {"P": (64, 300)})["P"]) <= 1e-5
elif case in ("gen_split", "gen_group"):
    import test_gpu_rule as T
    rows, n = (3, 70001) if case == "gen_split" else (5000, 48)
    d = T._row_reduce_dag(rows, n, T.DType.I32)
    x = port.Rng(905).tensor((rows, n), True)
    got, _ = run(d, {"X": dev(x, "f32")}, {"S": (rows,)})
    ok = np.array_equal(got["S"], oracle_eval(d, {"X": x}, {"S": (rows,)})["S"])
elif case == "maxpool":
    d = W.maxpool_dag(2, 16, 13)
    x = port.Rng(906).tensor((2, 16, 13, 13), True)
    got, _ = run(d, {"X": dev(x, "bf16", "cl")}, {"Y": (2, 16, 7, 7)})
    ok = np.array_equal(got["Y"], oracle_eval(d, {"X": x}, {"Y": (2, 16, 7, 7)})["Y"])
else:  # residual-before-ReLU conv epilogue (compact drain), plain and split-K 2
    L = W.ConvLayer("t", 64, 14, 256, 1, 1, 0, 1)
    d = W.conv_bn_dag(L, 2, residual=True)
    rng = port.Rng(907)
    ins = {"X": rng.tensor((2, 64, 14, 14), True), "W": rng.tensor((256, 64, 1, 1), True),
           "Scale": rng.tensor((256,), True), "Shift": rng.tensor((256,), True), "R": rng.tensor((2, 256, 14, 14), True)}
    t = {k: dev(v, "bf16", "cl" if v.ndim == 4 else None) for k, v in ins.items()}
    z = torch.empty((2, 256, 14, 14), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    from paper_2210_09603_b200 import Plan
    ex = Plan(d, ScheduleConfig(block_n=256, split_k=2 if case == "res_sk2" else 1)).bind([t[n] for n in d.inputs], [z])
    ex.launch(); torch.cuda.synchronize()
    want = port.round_bf16(oracle_eval(d, ins, {"Z": (2, 256, 14, 14)})["Z"])  # the bf16 store rounds
    ok = np.array_equal(z.float().cpu().numpy(), want)
print(case, "equal" if ok else "DIFF")
PY
for tool in memcheck racecheck synccheck; do
  for c in gen_softmax interp_softmax gen_split gen_group maxpool res res_sk2; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python $OUT/cases.py $c > $OUT/${tool}_${c}.log 2>&1
    echo "exit $?" >> $OUT/${tool}_${c}.log
  done
done
grep -h -E "ERROR SUMMARY|equal|DIFF|^exit" $OUT/*.log | sort | uniq -c
