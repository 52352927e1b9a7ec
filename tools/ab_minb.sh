#!/bin/bash
# fused GMRES occupancy A/B on the C4 steady state: 2 CTAs/SM (default) vs 3 (GF_MINB=3, G=444)
for v in "|" "-DGF_MINB=3|444" "-DGF_MINB=3|296"; do
  f="${v%%|*}"; g="${v##*|}"
  TT_NVCC_EXTRA="$f" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== flags '$f' grid '$g'"
  if [ -n "$g" ]; then export TT_GF_GRID=$g; else unset TT_GF_GRID; fi
  timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|gm_chunk_kernelILb0"
done
