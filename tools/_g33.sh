mkdir -p gpurun_out
GTS_STREAM_TRACE=1 GTS_TRACE=1 timeout 900 python bench.py --workload dna_stream --no-cpu-baseline > gpurun_out/bench_dna_stream_g33.json 2> gpurun_out/bench_dna_stream_g33.err
timeout 600 python -m pytest tests -m gpu -x -q -k "stream" > gpurun_out/pytest_gpu_g33.log 2>&1; echo pytest=$? > gpurun_out/status_g33.txt
echo done >> gpurun_out/status_g33.txt
