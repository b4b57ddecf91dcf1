#!/bin/bash
# One `ncu --set full` capture per kernel family the bench (and config 1) launches,
# into gpurun_out/ncu_r02/ (summarised into profiles/ by scripts/ncu_table.py).
OUT=gpurun_out/ncu_r02
mkdir -p $OUT
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name, kernel regex, skip, command...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 300 $NCU -k regex:$re -s $skip -c 1 -o $OUT/$name "$@" > $OUT/$name.log 2>&1
}
cap conv1_rowband rowband 3 python scripts/run_case.py --case conv:conv1 --iters 2
cap l1c2_bn96 tm_gemm 3 python scripts/run_case.py --case conv:l1.c2 --bn 96 --raster 1 --iters 2
cap l2c2_bn128 tm_gemm 3 python scripts/run_case.py --case conv:l2.c2 --bn 128 --iters 2
cap l3c2_bn96 tm_gemm 3 python scripts/run_case.py --case conv:l3.c2 --bn 96 --raster 1 --iters 2
cap l1c3_bn256 tm_gemm 3 python scripts/run_case.py --case conv:l1.c3 --bn 256 --iters 2
cap l4c3_bn192 tm_gemm 3 python scripts/run_case.py --case conv:l4.c3 --bn 192 --iters 2
cap l4c2_bn128sk2 tm_gemm 3 python scripts/run_case.py --case conv:l4.c2 --bn 128 --sk 2 --iters 2
cap ffn_gemm1_pair256 tm_gemm 6 python scripts/run_case.py --case ffn --bm 256 --bn 256 --iters 2
cap ffn_gemm2_pair256 tm_gemm 7 python scripts/run_case.py --case ffn --bm 256 --bn 256 --iters 2
cap attn_qk tm_gemm 3 python scripts/run_case.py --case qk --bn 128 --iters 2
cap attn_pv tm_gemm 3 python scripts/run_case.py --case pv --bn 64 --iters 2
cap l1c2_halo halo 3 python scripts/run_case.py --case conv:l1.c2 --math halo --iters 2
cap l2c2_halo halo 3 python scripts/run_case.py --case conv:l2.c2 --math halo --iters 2
cap l3c2_halo halo 3 python scripts/run_case.py --case conv:l3.c2 --math halo --iters 2
cap config1_simt simt 2 python scripts/ncu_cases.py simt
cap config1_tf32 tm_gemm 2 python scripts/ncu_cases.py tf32
cap softmax_reduce rule_tree 2 python scripts/ncu_cases.py softmax
cap softmax_rule rule_elem 2 python scripts/ncu_cases.py softmax
# text summaries on the box (the .ncu-rep files are too large to bring back)
python scripts/ncu_table.py $OUT/*.ncu-rep > $OUT/table.md 2> $OUT/table.err
for r in $OUT/*.ncu-rep; do
  n=$(basename $r .ncu-rep)
  ncu -i $r --page details > $OUT/$n.details.txt 2>/dev/null
  python scripts/ncu_lines.py $r 20 > $OUT/$n.lines.txt 2>/dev/null
done
mkdir -p $OUT/keep; for k in conv1_rowband l3c2_halo; do mv $OUT/$k.ncu-rep $OUT/keep/ 2>/dev/null; done
rm -f $OUT/*.ncu-rep
du -sh $OUT
