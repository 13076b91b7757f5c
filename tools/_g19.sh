mkdir -p gpurun_out
for i in 1 2; do timeout 300 python tools/step_trace.py > gpurun_out/steptrace_g19_$i.txt 2>&1; done
for mode in none off full off; do GTS_CLOCK_MODE=$mode timeout 300 python bench.py --workload words --steps 12 --no-cpu-baseline > gpurun_out/bench_words_g19_$mode.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_words_g19_$mode.json').read().strip().splitlines()[-1]);print('$mode',d['step_ms'])" >> gpurun_out/steps_g19.txt; done
echo done > gpurun_out/status_g19.txt
