#!/bin/bash
tag=${1:-m}
out=gpurun_out; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_mma -s 3 -c 1 \
    -o $out/prof_mma_$tag python bench.py --workload vec128 --n 200000 --nq 20000 --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_mma_stdout_$tag.txt 2>&1
