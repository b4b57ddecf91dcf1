#!/bin/bash
# round-2 probe 1: GPU suite + hang probes of the schedules excluded in round 1
OUT=gpurun_out/r02p1
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
for pdl in 0 1; do
  for case in ffn gelu res; do
    if [ $pdl = 1 ]; then export TMB_PDL=1; else unset TMB_PDL; fi
    timeout 300 python scripts/hang_probe.py --case $case --reps 30 \
      --cfgs pair128,pair128sk2,bn64sk2,bn64sk2db,sk4,bn256sk4,bn128sk2,bn192sk2,pair256,pair256sk2,pair64 \
      > $OUT/hang_${case}_pdl$pdl.log 2>&1; echo "exit $?" >> $OUT/hang_${case}_pdl$pdl.log
  done
done
echo done > $OUT/DONE
