#!/bin/bash
# A/B of env assignments on one bench config: gpurun -- bash tools/gpu_ab_cfg.sh <tag> <config> "" "X=1" ...
set -u
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
i=0
for envs in "$@"; do
  env $envs timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e > $OUT/bench_$i.log 2>&1
  echo "$envs" > $OUT/bench_$i.env
  i=$((i+1))
done
