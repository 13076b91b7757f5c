mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g15.log 2>&1; echo pytest=$? > gpurun_out/status_g15.txt
timeout 900 python bench.py --workload l1shard --no-cpu-baseline > gpurun_out/bench_l1shard_g15.json 2>&1
timeout 400 python bench.py --workload vec128 --no-cpu-baseline > gpurun_out/bench_vec128_g15.json 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_tile -s 20 -c 1 -o gpurun_out/prof_l1shard_g15 -f python bench.py --workload l1shard --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l1shard_g15.log 2>&1
echo done >> gpurun_out/status_g15.txt
