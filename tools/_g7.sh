mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g7.log 2>&1; echo pytest=$? > gpurun_out/status_g7.txt
timeout 400 python bench.py --workload vec128 --no-cpu-baseline > gpurun_out/bench_vec128_g7.json 2>&1
timeout 300 python bench.py --workload words --steps 10 --no-cpu-baseline > gpurun_out/bench_words_g7.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_mma2 -s 6 -c 1 -o gpurun_out/prof_vec128_g7 -f python bench.py --workload vec128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_vec128_g7.log 2>&1
timeout 900 python bench.py --workload l1shard --no-cpu-baseline > gpurun_out/bench_l1shard_g7.json 2>&1
echo done >> gpurun_out/status_g7.txt
