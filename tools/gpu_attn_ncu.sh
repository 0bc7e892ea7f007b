#!/bin/bash
# Attention: parity tests, bench phases, and one ncu --set full capture (source counters) of
# attn_tc_kernel on the config-C layer probe.
OUT=gpurun_out/${1:-attnncu}; mkdir -p $OUT
[ -z "$NOTEST" ] && timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_llava.py tests/test_gpu_parity.py -m gpu -x -q -k "attention or config_c_depth or config_a or request or link" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
[ -z "$NOTEST" ] && timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench.log 2>&1
MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py C > $OUT/ts_C.log 2>&1
[ -n "$NCU" ] && timeout 400 ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 5 -c 1 -o $OUT/attn_C python tools/attn_probe.py C > $OUT/ncu.log 2>&1
MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py pair > $OUT/ts_pair.log 2>&1
MPIC_ATTN_TS=1 timeout 60 python tools/attn_probe.py single > $OUT/ts_single.log 2>&1
