#!/bin/bash
OUT=gpurun_out/r02p5
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tuner.py tests/test_gpu_robustness.py tests/test_gpu_baseline_shapes.py -q > $OUT/pytest_new.log 2>&1; echo "exit $?" >> $OUT/pytest_new.log
for c in "gemm:1024,1024,1024 --bn 128" "conv:l3.c3 --bn 192" "conv:l4.c1 --bn 64"; do
  set -- $c
  n=$(echo $1 | tr ':,' '__')
  timeout 120 python scripts/run_case.py --case $1 $2 $3 --gap > $OUT/gap_$n.log 2>&1
  timeout 120 python scripts/run_case.py --case $1 $2 $3 --trace > $OUT/trace_$n.log 2>&1
  TMB_NO_PDL=1 timeout 120 python scripts/run_case.py --case $1 $2 $3 --gap > $OUT/gap_nopdl_$n.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tm_gemm --csv python scripts/run_case.py --case $1 $2 $3 --iters 5 > $OUT/ncu_$n.csv 2>&1
done
echo done > $OUT/DONE
