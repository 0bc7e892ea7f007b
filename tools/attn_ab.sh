#!/bin/bash
# A/B of two attention builds (default lib vs paper_2502_01960_b200/lib_old) with per-CTA spans.
OUT=gpurun_out/${1:-attnab}; mkdir -p $OUT
for v in new old; do
  if [ $v = old ]; then export MPIC_B200_LIB=$PWD/paper_2502_01960_b200/lib_old/libmpic_b200.so; fi
  timeout 60 python tools/attn_probe.py C pair single > $OUT/probe_$v.log 2>&1
  MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py pair > $OUT/ts_pair_$v.log 2>&1
  MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py C > $OUT/ts_C_$v.log 2>&1
done
