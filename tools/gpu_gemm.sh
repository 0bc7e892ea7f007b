#!/bin/bash
# GEMM iteration: GEMM parity tests + LLaVA parity + bench phases (config C and B).
OUT=gpurun_out/${1:-gemm}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_llava.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench_0.log 2>&1; echo "C" > $OUT/bench_0.env
timeout 200 python bench.py --config B --no-cpu-baseline --no-e2e --no-serving --steps 10 > $OUT/bench_1.log 2>&1; echo "B" > $OUT/bench_1.env
