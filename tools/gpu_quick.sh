#!/bin/bash
# Quick GPU check: parity tests + one config C bench line (no CPU baseline).
# Usage: gpurun --timeout 1200 -- bash tools/gpu_quick.sh <tag> [extra bench args]
set -u
TAG=${1:-quick}; shift || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline "$@" > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
echo done > $OUT/DONE
