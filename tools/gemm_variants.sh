#!/bin/bash
# GEMM variant comparison on the projection shapes (diagnostics)
cd "$(dirname "$0")/.."
for v in auto tok sk; do
  echo "== MPIC_GEMM_VARIANT=$v"
  if [ "$v" = auto ]; then python tools/gemm_probe.py 2>&1 | head -5; else MPIC_GEMM_VARIANT=$v python tools/gemm_probe.py 2>&1 | head -5; fi
done
