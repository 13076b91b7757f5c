mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_g31.log 2>&1; echo pytest=$? > gpurun_out/status_g31.txt
echo done >> gpurun_out/status_g31.txt
