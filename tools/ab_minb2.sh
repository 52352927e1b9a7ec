#!/bin/bash
# A/B: CTAs per SM of the fused GMRES kernel (register cap 168 / 128) on the C4 steady state
for cfg in "3 444" "4 592"; do
  set -- $cfg
  TT_NVCC_EXTRA="-DGF_MINB=$1" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== GF_MINB=$1 grid $2"
  TT_GF_GRID=$2 timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused|^ +(8|10|19|24) +[0-9.]+ +[0-9.]+ +4.0"
done
