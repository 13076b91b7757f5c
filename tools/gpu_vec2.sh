#!/bin/bash
tag=${1:-v}
out=gpurun_out; mkdir -p $out
(timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -15) > $out/pytest_gpu_$tag.log
GTS_TRACE=1 timeout 600 python bench.py --workload vec128 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_vec128_$tag.json 2> $out/trace_vec128_$tag.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_mma -s 3 -c 1 \
    -o $out/prof_mma_$tag python bench.py --workload vec128 --n 200000 --nq 20000 --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_mma_stdout_$tag.txt 2>&1
