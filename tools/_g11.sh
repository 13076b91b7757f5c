mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g11.log 2>&1; echo pytest=$? > gpurun_out/status_g11.txt
timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g11.json 2> gpurun_out/bench_words_g11.err
timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g11b.json 2> gpurun_out/bench_words_g11b.err
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g11.json 2> gpurun_out/bench_dna_g11.err
timeout 400 python bench.py --workload vec128 --no-cpu-baseline > gpurun_out/bench_vec128_g11.json 2>&1
echo done >> gpurun_out/status_g11.txt
