mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_g17.txt 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "edit or words or dna or string or golden or reference" > gpurun_out/pytest_gpu_g17.log 2>&1; echo pytest=$? > gpurun_out/status_g17.txt
for mode in none full none full; do GTS_CLOCK_MODE=$mode timeout 300 python bench.py --workload words --steps 12 --no-cpu-baseline > gpurun_out/bench_words_g17_$mode.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_words_g17_$mode.json').read().strip().splitlines()[-1]);print('$mode',d['step_ms'])" >> gpurun_out/steps_g17.txt; done
GTS_EDIT_CLAIM=16 timeout 300 python bench.py --workload words --no-cpu-baseline > gpurun_out/bench_words_g17_claim16.json 2>&1
timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g17.json 2>&1
GTS_EDIT_CLAIM=16 timeout 300 python bench.py --workload dna --no-cpu-baseline > gpurun_out/bench_dna_g17_claim16.json 2>&1
echo done >> gpurun_out/status_g17.txt
