#!/bin/bash
OUT=gpurun_out/exp8; mkdir -p $OUT
TMB_DBG=3 timeout 120 python scripts/run_case.py --case gemm:18944,256,2304 --bm 256 --bn 128 --bt --trace > $OUT/t_dbg3.txt 2>&1
timeout 120 python scripts/run_case.py --case gemm:18944,256,2304 --bm 256 --bn 128 --bt --trace > $OUT/t.txt 2>&1
TMB_DBG=3 timeout 120 python scripts/run_case.py --case gemm:18944,256,2304 --bm 128 --bn 256 --bt --trace > $OUT/t_dbg3_cg1.txt 2>&1
timeout 120 python scripts/run_case.py --case gemm:8192,8192,8192 --bm 256 --bn 256 --trace > $OUT/t_big.txt 2>&1
