#!/bin/bash
# The round's measurement set, run on the GPU box under gpurun:
#   tools/round_profile.sh <tag>
# pytest -m gpu, smoke(), bench lines of every workload (with CPU baselines),
# ncu launch lists + one --set full capture of the dominant kernel for words,
# vec128 and l1shard, the reference arm.  Summaries: tools/ncu_summary.py and
# tools/bench_table.py -> profiles/.
set -u
T=${1:-rXX}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo pytest=$? > gpurun_out/status_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke=$? >> gpurun_out/status_$T.txt
tools/gpu_profile.sh words $T k_leaf_edit 2
tools/gpu_profile.sh vec128 $T k_leafgroup_mma2 6
for w in tloc dna; do timeout 600 python bench.py --workload $w > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err; done
timeout 900 python bench.py --workload l1shard > gpurun_out/bench_l1shard_$T.json 2> gpurun_out/bench_l1shard_$T.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_tile -s 20 -c 1 -o gpurun_out/prof_l1shard_$T -f python bench.py --workload l1shard --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l1shard_$T.log 2>&1
timeout 900 python bench.py --workload dna_stream > gpurun_out/bench_dna_stream_$T.json 2> gpurun_out/bench_dna_stream_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_words_$T.json 2> gpurun_out/bench_ref_words_$T.err
echo done >> gpurun_out/status_$T.txt
