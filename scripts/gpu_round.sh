#!/bin/bash
# One gpurun call's worth of evidence: GPU parity tests, smoke, both bench arms,
# the ncu launch list of the bench command and one full capture of a conv kernel.
#   gpurun --timeout 3000 -- bash scripts/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu >> $OUT/nproc.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py --per-item > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
cp tuning_cache.json $OUT/tuning_cache.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --tune off --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tm_gemm -s 5 -c 2 \
    -o $OUT/conv_l3c2 python scripts/run_case.py --case conv:l3.c2 --iters 8 > $OUT/ncu_full_conv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tm_gemm -s 5 -c 2 \
    -o $OUT/ffn python scripts/run_case.py --case ffn --iters 8 > $OUT/ncu_full_ffn.log 2>&1
echo done > $OUT/DONE
