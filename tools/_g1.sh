mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g1.log 2>&1; echo pytest=$? > gpurun_out/status_g1.txt
for mode in full clock none; do GTS_CLOCK_MODE=$mode timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g1_$mode.json 2>&1; done
GTS_NO_GROUPED=1 timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g1_rowwise.json 2>&1
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g1.json 2>&1
echo done >> gpurun_out/status_g1.txt
