#!/bin/bash
# Quick A/B of the current build on the GPU box: GEMM-heavy parity tests, the C4
# steady-state probe (tools/probe_c4.py 8 2) and the C5 double sweep at r = 64/128/256.
python -m pytest tests/test_gpu_sweep.py tests/test_gpu_structured.py tests/test_gpu_tt.py tests/test_gpu_tsqr.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused|us  |^ +[0-9]+ +[0-9.]+ +[0-9.]+ +4.0" | head -48
for r in 64 128 256; do
  python bench.py --workload c5 --rank $r --steps 10 --warmup 3 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('c5 r=$r', round(d['value'], 1), d['unit'], d.get('contraction_pct_dmma_peak', d.get('roofline', {}).get('frac')))
"
done
