#!/bin/bash
# Attention quick check: probes (20 s each, hang-safe) then TS timelines.
OUT=gpurun_out/${1:-aq}; mkdir -p $OUT
for c in single pair C; do timeout 20 python tools/attn_probe.py $c >> $OUT/probe.log 2>&1; echo "$c exit $?" >> $OUT/probe.log; done
grep -q "exit 124" $OUT/probe.log && exit 0
for c in single pair C; do MPIC_ATTN_TS=1 timeout 30 python tools/attn_probe.py $c > $OUT/ts_$c.log 2>&1; done
