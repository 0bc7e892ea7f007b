set -u
O=gpurun_out/r2t; mkdir -p $O
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --config B --no-cpu-baseline > $O/bench_B.log 2>&1
timeout 600 python bench.py --config A --no-cpu-baseline > $O/bench_A.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
bash tools/gpu_prof.sh r2t 'tc_pgemm|attn_tc|assemble' 400 6
