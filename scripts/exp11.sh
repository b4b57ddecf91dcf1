#!/bin/bash
OUT=gpurun_out/exp11; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q -k "small_channel or conv" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for s in 0 2 4; do timeout 120 python scripts/run_case.py --case conv:conv1 --bn 64 --stages $s --iters 20 >> $OUT/conv1.txt 2>&1; done
timeout 120 python scripts/run_case.py --case conv:conv1 --bn 64 --trace > $OUT/trace_conv1.txt 2>&1
