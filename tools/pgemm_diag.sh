#!/bin/bash
# Time decomposition of the pair GEMM on the projection shapes (diagnostics).
cd "$(dirname "$0")/.."
for grp in 512 256; do
  for dbg in 0 1 9 2 4 6 8; do
    echo "== MPIC_PG_GROUP=$grp MPIC_PG_DBG=$dbg (1 no epilogue, 2 no X loads, 4 no W loads, 8 no MMA)"
    MPIC_PG_GROUP=$grp MPIC_PG_DBG=$dbg python tools/gemm_probe.py 2>&1 | head -4
  done
done
