#!/bin/bash
# A/B of the QR kernel's thread count on the C4 steady state (tools/probe_c4.py 8 2)
for v in "$@"; do
  TT_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== variant '$v'"
  timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|qr_kernel|jacobi_cluster"
done
