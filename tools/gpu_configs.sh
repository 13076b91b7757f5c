#!/bin/bash
# Every BASELINE config on the current build (bench lines for the record)
tag=${1:-c}
out=gpurun_out; mkdir -p $out
timeout 900 python bench.py --workload dna_stream --steps 3 --warmup 2 > $out/bench_dna_stream_$tag.json 2> $out/err_dna_stream_$tag.txt
timeout 900 python bench.py --workload l1shard --steps 2 --warmup 3 > $out/bench_l1shard_$tag.json 2> $out/err_l1shard_$tag.txt
timeout 900 python bench.py --workload vec128 --steps 3 --warmup 3 > $out/bench_vec128_$tag.json 2> $out/err_vec128_$tag.txt
timeout 900 python bench.py --workload dna --steps 3 --warmup 3 > $out/bench_dna_$tag.json 2> $out/err_dna_$tag.txt
