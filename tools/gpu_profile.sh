#!/bin/bash
# Run on the GPU box (under gpurun): bench line + ncu launch list + one
# --set full capture of the top kernel for one workload.
#   tools/gpu_profile.sh <workload> <tag> <kernel-regex> [skip-launches]
set -u
W=$1; TAG=$2; K=$3; SKIP=${4:-2}
mkdir -p gpurun_out
timeout 600 python bench.py --workload $W > gpurun_out/bench_${W}_${TAG}.json 2> gpurun_out/bench_${W}_${TAG}.err
echo "bench_${W}=$?" >> gpurun_out/status_${TAG}.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${W}_${TAG}.csv \
    python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo "launches_${W}=$?" >> gpurun_out/status_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o gpurun_out/prof_${W}_${TAG} -f \
    python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_${W}_${TAG}.log 2>&1
echo "ncu_${W}=$?" >> gpurun_out/status_${TAG}.txt
tools/ncu_shrink.sh gpurun_out/prof_${W}_${TAG}.ncu-rep
