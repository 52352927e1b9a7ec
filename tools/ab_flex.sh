#!/bin/bash
# A/B of the flexible streamed tiles of the fused GMRES kernel on the C4 steady
# state (tools/probe_c4.py 8 2): pipeline slots and cost-model constants.
for v in "$@"; do
  TT_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== variant '$v'"
  timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused|^ +(8|10|19|24) +[0-9.]+ +[0-9.]+ +4.0"
done
