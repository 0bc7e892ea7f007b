#!/bin/bash
# A/B: GPU parity tests, then config C bench under each env assignment given (one per arg).
# Usage: gpurun --timeout 1500 -- bash tools/gpu_ab.sh <tag> "" "MPIC_X=1" ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
i=0
for envs in "$@"; do
  env $envs timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_$i.log 2>&1
  echo "$envs" > $OUT/bench_$i.env
  i=$((i+1))
done
echo done > $OUT/DONE
