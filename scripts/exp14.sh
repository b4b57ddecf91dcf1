#!/bin/bash
OUT=gpurun_out/${1:-exp14}; rm -rf $OUT; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q > $OUT/pytest.log 2>&1
for c in "conv:conv1 --bn 64" "conv:l3.c2 --bn 128" "conv:l3.c2 --bm 256 --bn 128" "conv:l1.c2 --bn 64" "gemm:8192,3072,768 --bn 256 --bm 256" "gemm:8192,8192,8192 --bn 256 --bm 256"; do
  timeout 120 python scripts/run_case.py --case $c --iters 10 >> $OUT/t.txt 2>&1
done
timeout 120 python scripts/run_case.py --case conv:l3.c2 --bm 256 --bn 128 --trace > $OUT/trace_l3c2.txt 2>&1
