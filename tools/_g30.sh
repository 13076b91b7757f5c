mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01h.log 2>&1; echo pytest=$? > gpurun_out/status_r01h.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01h.log 2>&1; echo smoke=$? >> gpurun_out/status_r01h.txt
tools/gpu_profile.sh words r01h k_leaf_edit 2
tools/gpu_profile.sh vec128 r01h k_leafgroup_mma2 6
for w in tloc dna; do timeout 600 python bench.py --workload $w > gpurun_out/bench_${w}_r01h.json 2> gpurun_out/bench_${w}_r01h.err; done
timeout 900 python bench.py --workload l1shard > gpurun_out/bench_l1shard_r01h.json 2> gpurun_out/bench_l1shard_r01h.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_tile -s 20 -c 1 -o gpurun_out/prof_l1shard_r01h -f python bench.py --workload l1shard --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l1shard_r01h.log 2>&1
timeout 900 python bench.py --workload dna_stream > gpurun_out/bench_dna_stream_r01h.json 2> gpurun_out/bench_dna_stream_r01h.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_words_r01h.json 2> gpurun_out/bench_ref_words_r01h.err
echo done >> gpurun_out/status_r01h.txt
