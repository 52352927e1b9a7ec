#!/bin/bash
# A/B of the fused GMRES kernel's GEMM tile pipeline on the C4 steady state
# (tools/probe_c4.py 8 2): default (BK 16, 2 stages) vs TT_NVCC_EXTRA variants.
for v in "" "-DGF_BK=32" "-DGF_ST=3" "-DGF_BK=32 -DGF_ST=3"; do
  TT_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== variant '$v'"
  timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused|gm_chunk_kernelILb0"
done
