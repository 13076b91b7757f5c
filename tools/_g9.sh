mkdir -p gpurun_out
tools/gpu_profile.sh words r01f k_leaf_edit 2
tools/gpu_profile.sh vec128 r01f k_leafgroup_mma2 6
for w in tloc dna; do timeout 600 python bench.py --workload $w > gpurun_out/bench_${w}_r01f.json 2> gpurun_out/bench_${w}_r01f.err; done
timeout 900 python bench.py --workload l1shard > gpurun_out/bench_l1shard_r01f.json 2> gpurun_out/bench_l1shard_r01f.err
timeout 900 python bench.py --workload dna_stream > gpurun_out/bench_dna_stream_r01f.json 2> gpurun_out/bench_dna_stream_r01f.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_words_r01f.json 2> gpurun_out/bench_ref_words_r01f.err
echo done > gpurun_out/status_g9.txt
