#!/bin/bash
# One gpurun call: GPU parity tests, smoke, reference conformance suites, bench, ncu launch list.
# Usage (from this container): gpurun --timeout 2400 -- bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for t in oracle/_ref/conformance/test_*; do
  timeout 300 $t > $OUT/conf_$(basename $t).log 2>&1; echo "exit $?" >> $OUT/conf_$(basename $t).log
done
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
timeout 300 python bench.py --config B --no-cpu-baseline > $OUT/bench_B.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo done > $OUT/DONE
