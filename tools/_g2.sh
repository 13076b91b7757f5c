mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g2.log 2>&1; echo pytest=$? > gpurun_out/status_g2.txt
timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g2.json 2>&1
GTS_NO_GROUPED=1 timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g2_rowwise.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_edit -s 3 -c 1 -o gpurun_out/prof_words_g2 -f python bench.py --workload words --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_words_g2.log 2>&1
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g2.json 2>&1
echo done >> gpurun_out/status_g2.txt
