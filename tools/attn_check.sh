#!/bin/bash
# Attention: hang-safe probes, TS timelines, then the attention parity tests and a bench line.
OUT=gpurun_out/${1:-ac}; mkdir -p $OUT
bash tools/attn_quick.sh ${1:-ac}
grep -q "exit 124" $OUT/probe.log && exit 0
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_llava.py tests/test_gpu_parity.py -m gpu -x -q -k "attention or config_c_depth or config_a or request or link" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench.log 2>&1
