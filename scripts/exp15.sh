#!/bin/bash
OUT=gpurun_out/${1:-exp15}; rm -rf $OUT; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1
timeout 900 python bench.py --per-item --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
