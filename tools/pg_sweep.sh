# MPIC_PG_* knob sweep over tools/gemm_fixed_probe.py shapes (pass configs as args)
for cfg in "$@"; do
  env $cfg TAG="$cfg" timeout 120 python tools/gemm_fixed_probe.py 2>&1 | tail -1
done
