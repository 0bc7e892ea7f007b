#!/bin/bash
# Attention iteration: attention parity tests + LLaVA-width request parity + probe timings.
OUT=gpurun_out/${1:-attn}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_llava.py -m gpu -x -q -k "attention or config_c_depth or config_a" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 60 python tools/attn_probe.py C pair single E16 > $OUT/probe.log 2>&1
MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py pair > $OUT/ts_pair.log 2>&1
MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py single > $OUT/ts_single.log 2>&1
timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench.log 2>&1
