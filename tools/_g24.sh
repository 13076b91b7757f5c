mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g24.log 2>&1; echo pytest=$? > gpurun_out/status_g24.txt
timeout 300 python bench.py --workload words --steps 8 --no-cpu-baseline > gpurun_out/bench_words_g24.json 2>&1
GTS_EDIT_SMEM_TEXT=0 timeout 300 python bench.py --workload words --steps 8 --no-cpu-baseline > gpurun_out/bench_words_g24_notx.json 2>&1
timeout 300 python bench.py --workload vec128 --steps 6 --no-cpu-baseline > gpurun_out/bench_vec128_g24.json 2>&1
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g24.json 2>&1
echo done >> gpurun_out/status_g24.txt
