#!/bin/bash
OUT=gpurun_out/exp5; mkdir -p $OUT
for c in "conv:l3.c2 --bm 256 --bn 128" "conv:l1.c2 --bm 256 --bn 64" "gemm:8192,3072,768 --bn 256 --bm 256" "conv:l3.c1 --bn 128"; do
  echo "== $c" >> $OUT/times.txt
  timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
  TMB_DBG=3 timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
  TMB_DBG=2 timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
done
TMB_DBG=3 timeout 120 python scripts/run_case.py --case conv:l3.c2 --bm 256 --bn 128 --trace > $OUT/trace_l3c2_dbg3.txt 2>&1
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tmabench scripts/tmabench.cu -lcuda
for P in 1 2 4; do timeout 60 /tmp/tmabench 148 sweep 2 3 $P > $OUT/tb_P$P.txt 2>&1; done
