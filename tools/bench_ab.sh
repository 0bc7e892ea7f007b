#!/bin/bash
# A/B of env assignments on the config C bench (device legs only): bench_ab.sh <tag> "" "X=1" ...
OUT=gpurun_out/$1; shift; mkdir -p $OUT
i=0
for envs in "$@"; do
  env $envs timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench_$i.log 2>&1
  echo "$envs" > $OUT/bench_$i.env; i=$((i+1))
done
