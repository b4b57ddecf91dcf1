#!/bin/bash
# quick per-case timings (graph of 20 launches) + GPU parity
OUT=gpurun_out/${1:-exp2}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
for c in "gemm:8192,8192,8192 --bn 256 --bm 256" "gemm:8192,3072,768 --bn 256" "gemm:8192,3072,768 --bn 256 --bm 256" "gemm:8192,768,3072 --bn 256 --bm 256" "conv:l3.c2 --bm 256 --bn 128" "conv:l1.c2 --bm 256 --bn 64" "conv:l4.c2 --bm 256 --bn 128 --sk 2" "conv:l3.c1 --bn 128" "conv:l2.c3 --bn 192"; do
  echo "== $c" >> $OUT/times.txt
  timeout 120 python scripts/run_case.py --case $c --iters 20 >> $OUT/times.txt 2>&1
done
timeout 900 python bench.py --per-item --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 120 python scripts/run_case.py --case conv:l3.c2 --bm 256 --bn 128 --trace > $OUT/trace_l3c2.txt 2>&1
timeout 120 python scripts/run_case.py --case gemm:8192,3072,768 --bn 256 --bm 256 --trace > $OUT/trace_ffn1.txt 2>&1
