#!/bin/bash
# C5 double sweep: one stream vs applies on a side stream, r = 64 / 128 / 256
for r in 64 128 256; do
  for f in "--one-stream" ""; do
    python bench.py --workload c5 --rank $r --steps 10 --warmup 3 $f 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($r, '$f', round(d['value']), 'GFLOP/s', round(d['pct_dmma_peak'],1), '%', round(d['ms_per_step'],2), 'ms')"
  done
done
