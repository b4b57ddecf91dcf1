#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) on one small case of each
# kernel family added in round 2: the row-band stem conv, the halo conv, the
# cooperative split-K reduction, the rule-based / reduce kernels.
OUT=gpurun_out/san_r02
mkdir -p $OUT
cat > $OUT/cases.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
case = sys.argv[1]
if case == "rowband":
    import test_gpu_rowband as T
    got, want = T._run(1, 3, 64, 64, 7, 2, 3, cpad=4, seed=901)
elif case == "halo":
    import test_gpu_halo as T
    got, want = T._run(1, 64, 20, 64, 3, 1, seed=902)
elif case == "splitk":
    from paper_2210_09603_b200 import ScheduleConfig, workloads as W
    import test_gpu_baseline_shapes as T
    L = [x for x in W.RESNET50 if x.name == "l4.c2"][0]
    got, want = T._conv_case(L, 1, ScheduleConfig(block_n=256, split_k=4), seed=903)
elif case == "softmax":
    import test_gpu_rule as T
    d = T._softmax_dag(64, 300)
    from gpu_util import dev, run
    from oracle import port
    x = port.Rng(904).tensor((64, 300))
    got, _ = run(d, {"X": dev(x, "f32")}, {"P": (64, 300)})
    got, want = got["P"], got["P"]
print(case, "equal" if np.array_equal(got, want) else "DIFF")
PY
for tool in memcheck racecheck synccheck; do
  for c in rowband halo splitk softmax; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python $OUT/cases.py $c > $OUT/${tool}_${c}.log 2>&1
    echo "exit $?" >> $OUT/${tool}_${c}.log
  done
done
