#!/bin/bash
# A/B: when the stand-alone GEMM uses 32x32 tiles (less padding at ranks like 132) on the C4 steady state
for cfg in "256 296" "100000 296" "100000 600" "1024 296"; do
  set -- $cfg
  echo "== TT_GEMM_SMALL_K=$1 TT_GEMM_SMALL_T=$2"
  TT_GEMM_SMALL_K=$1 TT_GEMM_SMALL_T=$2 timeout 300 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|gemm_dmma_kernel|splitk"
done
