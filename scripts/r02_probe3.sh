#!/bin/bash
# round-2 probe 3: new gate / dag_eval / fp16 / robustness tests, full GPU suite, cold re-tune + bench
OUT=gpurun_out/r02p3
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tuner.py tests/test_gpu_robustness.py -q -x > $OUT/pytest_new.log 2>&1; echo "exit $?" >> $OUT/pytest_new.log
timeout 900 python -m pytest tests/test_gpu_gemm.py -q > $OUT/pytest_gemm.log 2>&1; echo "exit $?" >> $OUT/pytest_gemm.log
timeout 1500 python bench.py --tune auto --per-item > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
cp tuning_cache.json $OUT/tuning_cache.json
timeout 900 python -m pytest tests/test_gpu_baseline_shapes.py -q > $OUT/pytest_shapes.log 2>&1; echo "exit $?" >> $OUT/pytest_shapes.log
echo done > $OUT/DONE
