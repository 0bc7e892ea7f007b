#!/bin/bash
OUT=gpurun_out/${1:-cps}; mkdir -p $OUT
for c in 1 2 4 6; do MPIC_ATTN_CHUNKS_PER_SM=$c timeout 30 python tools/attn_probe.py C E16 >> $OUT/probe.log 2>&1; echo "cps $c exit $?" >> $OUT/probe.log; done
MPIC_ATTN_CHUNKS_PER_SM=2 timeout 120 compute-sanitizer --print-limit 5 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 1 --warmup 1 > $OUT/sanitizer.log 2>&1
