#!/bin/bash
# Runs the round's measurements on a GPU box; outputs under gpurun_out/r01/.
set -u
O=gpurun_out/r01
mkdir -p $O
timeout 900 python bench.py > $O/bench_c1_r01.json 2> $O/bench_c1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c1_r01.json 2> $O/bench_ref.err
timeout 900 python bench.py --workload c2 --steps 5 --warmup 3 > $O/bench_c2_r01.json 2> $O/bench_c2.err
for r in 64 128 256; do
  timeout 900 python bench.py --workload c5 --rank $r --steps 10 --warmup 3 > $O/bench_c5_r${r}_r01.json 2> $O/bench_c5_$r.err
done
timeout 1500 python bench.py --workload c3 --steps 3 --warmup 3 --outer 30 > $O/bench_c3_r01.json 2> $O/bench_c3.err
timeout 1800 python bench.py --workload c4 --steps 3 --warmup 3 --outer 10 > $O/bench_c4_r01.json 2> $O/bench_c4.err
if [ "${NCU:-1}" = "1" ]; then
  ncu --set full --import-source on --clock-control none -k regex:gm_chunk_kernel --launch-skip 10 -c 3 \
      -o $O/ncu_gm_chunk_c1 python tools/profile_c1.py --iters 2 > $O/ncu_gm.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:gemm_dmma --launch-skip 200 -c 3 \
      -o $O/ncu_gemm_c5_r128 python bench.py --workload c5 --rank 128 --no-graph --steps 1 --warmup 0 > $O/ncu_c5.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:matvec_batched -c 1 \
      -o $O/ncu_mv_b64 python tools/probe_mv.py 64 2 > $O/ncu_mv.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:qr_kernel --launch-skip 200 -c 2 \
      -o $O/ncu_qr_c1 python tools/profile_c1.py --iters 2 > $O/ncu_qr.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 6000 --csv \
      --log-file $O/launches_c1.csv python tools/profile_c1.py --iters 6 > $O/ncu_l1.log 2>&1
  timeout 600 python tools/timeline.py c1 30 > $O/timeline_c1.txt 2>&1
  timeout 900 python tools/timeline.py c3 10 > $O/timeline_c3.txt 2>&1
fi
echo done
