#!/bin/bash
# Quick GPU check: parity tests + words bench (two clock-sampling intervals)
tag=${1:-q}
out=gpurun_out; mkdir -p $out
(timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15) > $out/pytest_gpu_$tag.log
(timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -2) > $out/bench_words_$tag.json
(timeout 900 python bench.py --no-cpu-baseline --clock-ms 2000 2>&1 | tail -2) > $out/bench_words_slowclk_$tag.json
