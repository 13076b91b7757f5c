mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g28.log 2>&1; echo pytest=$? > gpurun_out/status_g28.txt
timeout 900 python bench.py --workload l1shard --steps 3 --no-cpu-baseline > gpurun_out/bench_l1shard_g28.json 2>&1
timeout 300 python bench.py --workload tloc --no-cpu-baseline > gpurun_out/bench_tloc_g28.json 2>&1
timeout 300 python bench.py --workload vec128 --steps 6 --no-cpu-baseline > gpurun_out/bench_vec128_g28.json 2>&1
echo done >> gpurun_out/status_g28.txt
