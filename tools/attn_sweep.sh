#!/bin/bash
# Attention diagnostics: plan granularity sweep on the config-C layer + steady-state cases.
OUT=gpurun_out/${1:-attn}; mkdir -p $OUT
for c in 1 2 3 4 6; do MPIC_ATTN_CHUNKS_PER_SM=$c timeout 120 python tools/attn_probe.py C pair single; done > $OUT/sweep.log 2>&1
MPIC_ATTN_TS=1 timeout 120 python tools/attn_probe.py C > $OUT/ts_C.log 2>&1
MPIC_ATTN_TS=1 timeout 120 python tools/attn_probe.py pair > $OUT/ts_pair.log 2>&1
MPIC_ATTN_TS=1 timeout 120 python tools/attn_probe.py single > $OUT/ts_single.log 2>&1
