#!/bin/bash
OUT=gpurun_out/r02p4
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tuner.py tests/test_gpu_robustness.py tests/test_gpu_baseline_shapes.py -q > $OUT/pytest_new.log 2>&1; echo "exit $?" >> $OUT/pytest_new.log
timeout 1500 python scripts/pretune_shards.py > $OUT/pretune.log 2>&1; echo "exit $?" >> $OUT/pretune.log
cp tuning_cache.json $OUT/tuning_cache.json
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
