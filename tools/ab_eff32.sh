#!/bin/bash
# A/B of the fused-GMRES stage tile model (GF_EFF32) on the C4 steady state (tools/probe_c4.py 8 2)
for e in ${@:-0.6 0.8 1.0}; do
  TT_NVCC_EXTRA="-DGF_EFF32=$e" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== GF_EFF32=$e"
  timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused|us  " | head -6
done
python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
