mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "edit or words or dna or string or golden or reference or stream" > gpurun_out/pytest_gpu_g32.log 2>&1; echo pytest=$? > gpurun_out/status_g32.txt
timeout 300 python bench.py --workload words --steps 8 --no-cpu-baseline > gpurun_out/bench_words_g32.json 2>&1
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g32.json 2>&1
timeout 900 python bench.py --workload dna_stream --no-cpu-baseline > gpurun_out/bench_dna_stream_g32.json 2>&1
echo done >> gpurun_out/status_g32.txt
