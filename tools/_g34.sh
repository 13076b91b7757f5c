mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g34.log 2>&1; echo pytest=$? > gpurun_out/status_g34.txt
GTS_STREAM_TRACE=1 GTS_TRACE=1 timeout 900 python bench.py --workload dna_stream --no-cpu-baseline > gpurun_out/bench_dna_stream_g34.json 2> gpurun_out/bench_dna_stream_g34.err
timeout 300 python bench.py --workload words --steps 8 --no-cpu-baseline > gpurun_out/bench_words_g34.json 2>&1
echo done >> gpurun_out/status_g34.txt
