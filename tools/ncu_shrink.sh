#!/bin/bash
# On the GPU box: turn an ncu report into compact CSVs (raw metrics page and
# per-line source/SASS page, gzipped) and delete the .ncu-rep, so
# gpurun_out/ stays under gpurun's 64 MiB copy-back limit.
#   tools/ncu_shrink.sh gpurun_out/prof_words_r02.ncu-rep
set -u
R=$1
[ -f "$R" ] || exit 0
B=${R%.ncu-rep}
ncu -i "$R" --page raw --csv 2>/dev/null | gzip -9 > "$B.raw.csv.gz"
ncu -i "$R" --page source --csv --print-source cuda,sass 2>/dev/null | gzip -9 > "$B.src.csv.gz"
rm -f "$R"
