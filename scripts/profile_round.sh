#!/bin/bash
# Evidence for profiles/: GPU tests, bench (both arms), the ncu launch list of the
# bench command, and full ncu captures of representative kernels.
#   gpurun --timeout 3000 -- bash scripts/profile_round.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out/$TAG; rm -rf $OUT; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 1200 python bench.py --per-item > $OUT/bench.json 2> $OUT/bench.err
cp tuning_cache.json $OUT/tuning_cache.json
timeout 900 python bench.py > $OUT/bench2.json 2> $OUT/bench2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:tm_gemm --csv --log-file $OUT/launches.csv \
    python bench.py --launch-list > $OUT/ncu_launch_bench.log 2>&1
for c in "conv:l3.c2 --bn 128" "conv:l1.c2 --bn 64" "conv:conv1 --bn 64" "ffn"; do
  n=$(echo $c | tr ':. -' '____' | cut -c1-20)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tm_gemm -s 3 -c 1 \
      -o $OUT/full_$n python scripts/run_case.py --case $c --iters 4 > $OUT/ncu_full_$n.log 2>&1
done
echo done > $OUT/DONE
