#!/bin/bash
# GMRES(m) restart length A/B on the C4 steady state
for m in 40 20 30 60; do
  echo "== restart $m"
  TT_RESTART=$m timeout 600 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|^fused"
done
