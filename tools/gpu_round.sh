#!/bin/bash
# One GPU session: tests, smoke, benches, ncu launch list + full capture.
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu_$tag.txt
(timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -30) > $out/pytest_gpu_$tag.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5) > $out/smoke_$tag.log
(timeout 900 python bench.py --workload tloc 2>&1 | tail -3) > $out/bench_tloc_$tag.json
(timeout 1200 python bench.py 2>&1 | tail -3) > $out/bench_words_$tag.json
(timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_words_$tag.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_launch_stdout_$tag.txt 2>&1)
(timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_edit -s 6 -c 1 \
    -o $out/prof_verify_words_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_full_stdout_$tag.txt 2>&1)
ls -la $out
