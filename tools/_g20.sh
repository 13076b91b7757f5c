mkdir -p gpurun_out
for mode in full full off full; do GTS_CLOCK_MODE=$mode timeout 300 python bench.py --workload words --steps 12 --no-cpu-baseline > gpurun_out/bench_words_g20_$mode.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_words_g20_$mode.json').read().strip().splitlines()[-1]);print('$mode',d['step_ms'], d['e2e']['ms_per_step'])" >> gpurun_out/steps_g20.txt; done
timeout 300 python bench.py --workload vec128 --steps 8 --no-cpu-baseline > gpurun_out/bench_vec128_g20.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_vec128_g20.json').read().strip().splitlines()[-1]);print('vec128',d['step_ms'], d['e2e']['ms_per_step'])" >> gpurun_out/steps_g20.txt
echo done > gpurun_out/status_g20.txt
