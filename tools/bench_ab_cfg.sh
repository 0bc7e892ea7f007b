#!/bin/bash
# A/B of env assignments on one config: bench_ab_cfg.sh <tag> <config> "" "X=1" ...
OUT=gpurun_out/$1; CFG=$2; shift 2; mkdir -p $OUT
i=0
for envs in "$@"; do
  env $envs timeout 200 python bench.py --config $CFG --no-cpu-baseline --no-e2e --no-serving --no-fp32-mode --decode-steps 0 --steps 10 > $OUT/bench_$i.log 2>&1
  echo "$CFG $envs" > $OUT/bench_$i.env; i=$((i+1))
done
