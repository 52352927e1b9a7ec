#!/bin/bash
# Runs the round's measurements on a GPU box; outputs under gpurun_out/r01/.
set -u
O=gpurun_out/r01
mkdir -p $O
python tools/peaks_fp64 > /dev/null 2>&1 || true
timeout 900 python bench.py > $O/bench_c1_r01.json 2> $O/bench_c1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c1_r01.json 2> $O/bench_ref.err
timeout 900 python bench.py --workload c2 --steps 5 --warmup 3 > $O/bench_c2_r01.json 2> $O/bench_c2.err
for r in 64 128 256; do
  timeout 900 python bench.py --workload c5 --rank $r --steps 10 --warmup 3 > $O/bench_c5_r${r}_r01.json 2> $O/bench_c5_$r.err
done
timeout 1500 python bench.py --workload c3 --steps 3 --warmup 3 --outer 30 > $O/bench_c3_r01.json 2> $O/bench_c3.err
echo done
