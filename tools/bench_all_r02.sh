#!/bin/bash
# Round-2 numbers of the non-default workloads (profiles/r02/bench_*_r02.json)
python bench.py --workload c1 --steps 5 --warmup 3 > gpurun_out/bench_c1_r02.log 2>&1
python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_r02.log 2>&1
python bench.py --workload c2 --steps 5 --warmup 3 > gpurun_out/bench_c2_r02.log 2>&1
for r in 64 128 256; do python bench.py --workload c5 --rank $r --steps 10 --warmup 3 > gpurun_out/bench_c5_r${r}_r02.log 2>&1; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02.log 2>&1
python tools/timeline.py c1 30 > gpurun_out/timeline_c1_r02.txt 2>&1
