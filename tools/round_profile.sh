#!/bin/bash
# The round's measurement set, run on the GPU box under gpurun:
#   tools/round_profile.sh <tag> [sections]
# sections (default all): tests words vec128 small l1 l1big sanitize ref
# pytest -m gpu, smoke(), bench lines of every workload (with CPU baselines),
# ncu launch lists + one --set full capture of the dominant kernel (and of
# the traversal kernel) per workload, compute-sanitizer on small cases, the
# reference arm.  Summaries: tools/ncu_summary.py and tools/bench_table.py
# -> profiles/.
set -u
T=${1:-rXX}
S=${2:-"tests words vec128 small l1 l1big sanitize ref"}
mkdir -p gpurun_out
has() { [[ " $S " == *" $1 "* ]]; }
st() { echo "$1=$2" >> gpurun_out/status_$T.txt; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; st pytest $?
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; st smoke $?
fi
if has words; then
  tools/gpu_profile.sh words $T k_leaf_edit 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expand -s 6 -c 1 \
      -o gpurun_out/prof_trav_words_$T -f python bench.py --workload words --steps 1 --warmup 1 --no-cpu-baseline \
      > gpurun_out/ncu_trav_words_$T.log 2>&1; st ncu_trav_words $?
  tools/ncu_shrink.sh gpurun_out/prof_trav_words_$T.ncu-rep
fi
if has vec128; then
  tools/gpu_profile.sh vec128 $T k_leafgroup_mma 6
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expand -s 20 -c 1 \
      -o gpurun_out/prof_trav_vec128_$T -f python bench.py --workload vec128 --steps 1 --warmup 1 --no-cpu-baseline \
      > gpurun_out/ncu_trav_vec128_$T.log 2>&1; st ncu_trav_vec128 $?
  tools/ncu_shrink.sh gpurun_out/prof_trav_vec128_$T.ncu-rep
fi
if has small; then
  for w in tloc dna; do timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err; st bench_$w $?; done
  timeout 900 python bench.py --workload dna_stream > gpurun_out/bench_dna_stream_$T.json 2> gpurun_out/bench_dna_stream_$T.err; st bench_dna_stream $?
fi
if has l1; then
  timeout 1200 python bench.py --workload l1shard > gpurun_out/bench_l1shard_$T.json 2> gpurun_out/bench_l1shard_$T.err; st bench_l1shard $?
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_leafgroup_tile -s 20 -c 1 \
      -o gpurun_out/prof_l1shard_$T -f python bench.py --workload l1shard --steps 1 --warmup 1 --no-cpu-baseline \
      > gpurun_out/ncu_l1shard_$T.log 2>&1; st ncu_l1shard $?
  tools/ncu_shrink.sh gpurun_out/prof_l1shard_$T.ncu-rep
fi
if has l1big; then
  timeout 2400 python bench.py --workload l1_100m --steps 3 --warmup 3 > gpurun_out/bench_l1_100m_$T.json 2> gpurun_out/bench_l1_100m_$T.err; st bench_l1_100m $?
fi
if has sanitize; then
  for tool in memcheck racecheck synccheck; do
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_paths.py \
        > gpurun_out/sanitize_${tool}_$T.log 2>&1; st sanitize_$tool $?
  done
fi
if has ref; then
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_words_$T.json 2> gpurun_out/bench_ref_words_$T.err; st ref $?
fi
echo done >> gpurun_out/status_$T.txt
