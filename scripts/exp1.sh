#!/bin/bash
OUT=gpurun_out/exp1; mkdir -p $OUT
for c in "gemm:8192,8192,8192 --bn 256" "gemm:8192,8192,8192 --bn 256 --bm 256" "gemm:8192,3072,768 --bn 256" "gemm:8192,3072,768 --bn 256 --bm 256" "conv:l3.c2 --bm 256 --bn 128" "conv:l3.c2 --bm 128 --bn 256" "conv:l1.c2 --bm 256 --bn 64"; do
  echo "== $c" >> $OUT/times.txt
  timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
done
timeout 120 python scripts/run_case.py --case gemm:8192,3072,768 --bn 256 --trace > $OUT/trace_ffn1.txt 2>&1
timeout 120 python scripts/run_case.py --case conv:l3.c2 --bm 256 --bn 128 --trace > $OUT/trace_l3c2.txt 2>&1
