#!/bin/bash
# Full GPU test suite, then bench A/B over env assignments (device legs only).
OUT=gpurun_out/$1; shift; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
i=0
for envs in "$@"; do
  env $envs timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench_$i.log 2>&1
  echo "$envs" > $OUT/bench_$i.env; i=$((i+1))
done
