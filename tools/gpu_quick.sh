#!/bin/bash
# Quick GPU check: parity tests + words bench (+ library trace) + ncu capture of the fused edit kernel
tag=${1:-q}
out=gpurun_out; mkdir -p $out
(timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15) > $out/pytest_gpu_$tag.log
GTS_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > $out/bench_words_$tag.json 2> $out/trace_words_$tag.txt
(timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_edit -s 6 -c 1 \
    -o $out/prof_leaf_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_full_stdout_$tag.txt 2>&1)
