#!/bin/bash
tag=${1:-p}
out=gpurun_out; mkdir -p $out
GTS_PHASES=1 GTS_TRACE=1 timeout 600 python bench.py --workload vec128 --n 300000 --nq 30000 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_vec128ph_$tag.json 2> $out/trace_vec128ph_$tag.txt
