#!/bin/bash
# ncu --set full captures of the top kernels of one bench step (1 GPU).
# Usage: gpurun --timeout 1800 -- bash tools/gpu_prof.sh <tag> [kernel-regex] [skip] [count]
set -u
TAG=${1:-prof}; RE=${2:-tc_gemm_sk|attn_tc}; SKIP=${3:-200}; CNT=${4:-6}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s $SKIP -c $CNT \
  -o $OUT/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
echo "ncu exit $?" >> $OUT/ncu.log
