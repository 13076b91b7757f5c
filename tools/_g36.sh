mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g36.log 2>&1; echo pytest=$? > gpurun_out/status_g36.txt
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g36.json 2>&1
timeout 900 python bench.py --workload dna_stream --no-cpu-baseline > gpurun_out/bench_dna_stream_g36.json 2>&1
timeout 300 python bench.py --workload words --steps 5 --no-cpu-baseline > gpurun_out/bench_words_g36.json 2>&1
echo done >> gpurun_out/status_g36.txt
