mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_vec -s 20 -c 1 -o gpurun_out/prof_l1shard_g13 -f python bench.py --workload l1shard --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l1shard_g13.log 2>&1
echo done > gpurun_out/status_g13.txt
