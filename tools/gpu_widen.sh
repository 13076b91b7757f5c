#!/bin/bash
# Other BASELINE configs on the current paths (bench lines for the record)
tag=${1:-w}
out=gpurun_out; mkdir -p $out
for wl in dna vec128; do
  GTS_TRACE=1 timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 > $out/bench_${wl}_$tag.json 2> $out/trace_${wl}_$tag.txt
done
GTS_TRACE=1 timeout 1200 python bench.py --workload l1shard --n 2000000 --nq 20000 --steps 3 --warmup 3 > $out/bench_l1shard_$tag.json 2> $out/trace_l1shard_$tag.txt
