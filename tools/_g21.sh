mkdir -p gpurun_out
GTS_TRACE=1 timeout 300 python bench.py --workload vec128 --steps 8 --no-cpu-baseline > gpurun_out/bench_vec128_g21.json 2> gpurun_out/bench_vec128_g21.err; python -c "import json;d=json.loads(open('gpurun_out/bench_vec128_g21.json').read().strip().splitlines()[-1]);print('vec128',d['step_ms'], d['e2e']['ms_per_step'])" >> gpurun_out/steps_g21.txt
timeout 300 python bench.py --workload vec128 --steps 8 --no-cpu-baseline > gpurun_out/bench_vec128_g21b.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_vec128_g21b.json').read().strip().splitlines()[-1]);print('vec128',d['step_ms'], d['e2e']['ms_per_step'])" >> gpurun_out/steps_g21.txt
echo done > gpurun_out/status_g21.txt
