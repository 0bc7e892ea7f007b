#!/bin/bash
# Attention A/B over several builds: tools/attn_libs.sh <tag> <libdir>... (default lib = "lib")
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for d in "$@"; do
  export MPIC_B200_LIB=$PWD/paper_2502_01960_b200/$d/libmpic_b200.so
  for c in C pair single; do MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py $c > $OUT/ts_${c}_$d.log 2>&1; done
  timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --no-fp32-mode --steps 10 > $OUT/bench_$d.log 2>&1
done
