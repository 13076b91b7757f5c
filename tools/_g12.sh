mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "tensor or mma or l2 or tloc or streaming" > gpurun_out/pytest_gpu_g12.log 2>&1; echo pytest=$? > gpurun_out/status_g12.txt
timeout 400 python bench.py --workload vec128 --no-cpu-baseline > gpurun_out/bench_vec128_g12.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_mma2 -s 6 -c 1 -o gpurun_out/prof_vec128_g12 -f python bench.py --workload vec128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_vec128_g12.log 2>&1
echo done >> gpurun_out/status_g12.txt
