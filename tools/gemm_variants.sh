#!/bin/bash
# C5 sweep GFLOP/s per DMMA GEMM variant (TT_GEMM_VARIANT)
for v in ${VARIANTS:-0 1}; do
  for r in 64 128 256; do
    TT_GEMM_VARIANT=$v timeout 200 python bench.py --workload c5 --rank $r --steps 5 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant', $v, 'r', $r, round(d['value']), 'GFLOP/s', round(d['pct_dmma_peak'],1), '%', round(d['ms_per_step'],2), 'ms')"
  done
done
