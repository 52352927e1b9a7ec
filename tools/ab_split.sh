#!/bin/bash
# split-K cap of the fused GMRES stage GEMMs (C4 steady state)
for v in "" "-DGF_MAXSPLIT=24" "-DGF_MAXSPLIT=32"; do
  TT_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g._build_module().build(force=True)" > /dev/null 2>&1
  echo "== '$v'"
  timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|gm_chunk_kernelILb0"
done
