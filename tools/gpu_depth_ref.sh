#!/bin/bash
# Parity depth sweep at config C (L' = 16, 32: GPU fp32/bf16 vs the reference vs fp64) and the
# reference's full 32-layer request time against the 2-layer sample the bench extrapolates.
OUT=gpurun_out/${1:-depth}; mkdir -p $OUT
timeout 600 python bench.py --cpu-leg --config C --layers-sample 32 --steps 1 --warmup 0 > $OUT/ref_full32.log 2>&1
timeout 300 python bench.py --cpu-leg --config C --layers-sample 2 --steps 2 --warmup 0 > $OUT/ref_sample2.log 2>&1
timeout 2400 python tools/depth_sweep.py --config C --depths 16 32 --out $OUT/depth_C.json > $OUT/depth.log 2>&1
echo done > $OUT/DONE
