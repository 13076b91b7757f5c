mkdir -p gpurun_out
GTS_TRACE=1 timeout 300 python tools/step_trace.py > gpurun_out/steptrace_g18.txt 2>&1
echo done > gpurun_out/status_g18.txt
