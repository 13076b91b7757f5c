mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g10.log 2>&1; echo pytest=$? > gpurun_out/status_g10.txt
GTS_TRACE=1 timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g10.json 2> gpurun_out/bench_words_g10.err
timeout 400 python bench.py --workload vec128 --no-cpu-baseline > gpurun_out/bench_vec128_g10.json 2>&1
GTS_TRACE=1 timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g10b.json 2> gpurun_out/bench_words_g10b.err
echo done >> gpurun_out/status_g10.txt
