#!/bin/bash
tag=${1:-v}
out=gpurun_out; mkdir -p $out
(timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15) > $out/pytest_gpu_$tag.log
GTS_TRACE=1 timeout 900 python bench.py --workload vec128 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_vec128_$tag.json 2> $out/trace_vec128_$tag.txt
GTS_TRACE=1 timeout 900 python bench.py --workload l1shard --n 2000000 --nq 20000 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_l1shard_$tag.json 2> $out/trace_l1shard_$tag.txt
