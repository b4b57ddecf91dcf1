#!/bin/bash
OUT=gpurun_out/exp7; mkdir -p $OUT
for c in "gemm:6272,256,2304 --bm 256 --bn 128 --bt" "gemm:6272,256,2304 --bm 256 --bn 128" "gemm:6272,256,2304 --bm 256 --bn 256 --bt" "gemm:6272,256,2304 --bm 256 --bn 256" "gemm:6272,256,2304 --bm 128 --bn 256 --bt" "gemm:6272,256,2304 --bm 128 --bn 128 --bt" "conv:l3.c2 --bm 256 --bn 256" "conv:l3.c2 --bm 128 --bn 256" "conv:l3.c2 --bm 128 --bn 128" "gemm:18944,256,2304 --bm 256 --bn 128 --bt" "gemm:18944,256,2304 --bm 256 --bn 256 --bt"; do
  echo "== $c" >> $OUT/times.txt
  timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
  TMB_DBG=3 timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
done
