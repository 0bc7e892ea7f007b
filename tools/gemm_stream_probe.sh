#!/bin/bash
# TMA streaming diagnostics of the 1-CTA tcgen05 GEMM (see tc_gemm.cu TcGemmArgs::dbg)
cd "$(dirname "$0")/.."
for dbg in 0 4 5 6 1 2; do
  echo "== MPIC_GEMM_NO_PAIR=1 MPIC_GEMM_DBG=$dbg (1 skip X, 2 skip W, 4 skip MMA)"
  MPIC_GEMM_NO_PAIR=1 MPIC_GEMM_DBG=$dbg python tools/gemm_probe.py 2>&1 | grep -v "^  " | head -5
done
