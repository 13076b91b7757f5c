mkdir -p gpurun_out
GTS_TRACE=1 timeout 300 python bench.py --workload vec128 --steps 8 --no-cpu-baseline > gpurun_out/bench_vec128_g22.json 2> gpurun_out/bench_vec128_g22.err; python -c "import json;d=json.loads(open('gpurun_out/bench_vec128_g22.json').read().strip().splitlines()[-1]);print('vec128 prime',d['step_ms'], d['e2e']['ms_per_step'], d['index_upload_s'])" >> gpurun_out/steps_g22.txt
GTS_POOL_PRIME_GB=0 timeout 300 python bench.py --workload vec128 --steps 8 --no-cpu-baseline > gpurun_out/bench_vec128_g22b.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_vec128_g22b.json').read().strip().splitlines()[-1]);print('vec128 noprime',d['step_ms'], d['e2e']['ms_per_step'], d['index_upload_s'])" >> gpurun_out/steps_g22.txt
echo done > gpurun_out/status_g22.txt
