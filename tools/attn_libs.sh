#!/bin/bash
# Attention A/B over several builds: tools/attn_libs.sh <tag> <libdir>... (default lib = "lib")
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for d in "$@"; do
  export MPIC_B200_LIB=$PWD/paper_2502_01960_b200/$d/libmpic_b200.so
  MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py C > $OUT/ts_C_$d.log 2>&1
  MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py pair > $OUT/ts_pair_$d.log 2>&1
  MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py single > $OUT/ts_single_$d.log 2>&1
  timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench_$d.log 2>&1
done
