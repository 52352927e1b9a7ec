#!/bin/bash
# A/B of the cluster size of the systolic Jacobi (TT_JC_CLUSTER) on the C4 steady state
for c in 0 6 11 8; do
  echo "== TT_JC_CLUSTER=$c"
  TT_JC_CLUSTER=$c timeout 300 python tools/probe_c4.py 8 2 c4 2>&1 | grep -E "^timed|jacobi_cluster"
done
timeout 200 python -m pytest tests/test_gpu_tt.py -x -q -m gpu 2>&1 | tail -2
