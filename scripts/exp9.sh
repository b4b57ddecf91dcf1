#!/bin/bash
OUT=gpurun_out/${1:-exp9}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 120 python scripts/run_case.py --case conv:conv1 --bn 64 --iters 20 > $OUT/conv1.txt 2>&1
timeout 120 python scripts/run_case.py --case conv:conv1 --bn 64 --stages 6 --iters 20 >> $OUT/conv1.txt 2>&1
timeout 1500 python bench.py --per-item --no-cpu-baseline --tune force > $OUT/bench.json 2> $OUT/bench.err
cp tuning_cache.json $OUT/tuning_cache.json
