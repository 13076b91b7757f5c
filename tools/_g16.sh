mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g16.log 2>&1; echo pytest=$? > gpurun_out/status_g16.txt
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g16.json 2>&1
timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g16.json 2>&1
timeout 900 python bench.py --workload l1shard --no-cpu-baseline > gpurun_out/bench_l1shard_g16.json 2>&1
echo done >> gpurun_out/status_g16.txt
