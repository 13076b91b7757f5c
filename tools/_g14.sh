mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g14.log 2>&1; echo pytest=$? > gpurun_out/status_g14.txt
timeout 900 python bench.py --workload l1shard --no-cpu-baseline > gpurun_out/bench_l1shard_g14.json 2>&1
timeout 300 python bench.py --workload tloc --no-cpu-baseline > gpurun_out/bench_tloc_g14.json 2>&1
echo done >> gpurun_out/status_g14.txt
