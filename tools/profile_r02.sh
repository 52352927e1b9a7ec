#!/bin/bash
# Round-2 evidence run (GPU box): the default bench line, then the ncu launch list
# of the timed step (NVTX range "timed") and ncu --set full captures of large
# fused-GMRES launches, QR and Jacobi launches inside the timed step.  ncu cannot
# profile kernel nodes of graphs with conditional nodes (graph mode 2), so the
# profiled runs use TT_NO_GRAPHS=1: the same kernels launched one by one.
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.log 2>&1
TT_NO_GRAPHS=1 python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/plain_r02.log 2>&1 && \
TT_NO_GRAPHS=1 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4_r02.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline \
    > gpurun_out/ncu_launch_r02.log 2>&1
TT_NO_GRAPHS=1 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:gm_chunk_kernelILb0 -s 40 -c 4 -o gpurun_out/prof_gm_c4_r02 \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_gm_r02.log 2>&1
TT_NO_GRAPHS=1 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
    -k regex:"qr_kernel|jacobi_cluster_kernel" -s 100 -c 4 -o gpurun_out/prof_qrsvd_c4_r02 \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_qrsvd_r02.log 2>&1
