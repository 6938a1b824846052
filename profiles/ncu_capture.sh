#!/bin/bash
# ncu capture recipe (run under gpurun on ONE B200, from the repo root).
#   profiles/ncu_capture.sh <config> <tag> <kernel-regex>
# 1) the plain command must exit 0 first; 2) launch list with per-launch device time;
# 3) one full-set capture of the top kernel.  Outputs land in gpurun_out/.
set -e
CFG=${1:-cfg2}
TAG=${2:-r01}
KRE=${3:-k_general_sort}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launches_${CFG}_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo "ncu done $CFG"
