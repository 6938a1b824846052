#!/bin/bash
# ncu evidence for one round (run under gpurun on ONE B200, from the repo root): per config, the
# plain command first, then an ncu launch list and one full-set capture of its dominant kernel,
# summarised on the box (the .ncu-rep files stay there: gpurun_out/ returns at most 64 MiB).
#   bash profiles/round_capture.sh <tag> [configs...]
set -u
TAG=${1:-r01}
shift || true
LIST=${*:-"cfg1:k_general_sort cfg1sw:k_short_wide32 cfg2:k_general_sort cfg2b:k_general_sort cfg3:k_tile_sort cfg4:k_permute cfg4s:k_permute cfg5:k_ms_scatter"}
mkdir -p gpurun_out/$TAG
cp profiles/traffic.json gpurun_out/$TAG/traffic.json 2>/dev/null
for a in $LIST; do
    c=${a%%:*}; k=${a##*:}
    if timeout 900 bash profiles/ncu_capture.sh $c $TAG $k; then
        rep=gpurun_out/prof_${c}_${TAG}.ncu-rep
        python profiles/ncu_summarize.py $rep 16 > gpurun_out/$TAG/summary_${c}.txt 2>&1
        python profiles/ncu_lines.py $rep 30 > gpurun_out/$TAG/lines_${c}.txt 2>&1
        ncu -i $rep --page details --csv > gpurun_out/$TAG/details_${c}.csv 2>/dev/null
        TRAFFIC_JSON=gpurun_out/$TAG/traffic.json python profiles/ncu_summarize.py --traffic $c=$rep \
            --source-dir profiles/$TAG > /dev/null 2>&1
        mv gpurun_out/launches_${c}_${TAG}.csv gpurun_out/$TAG/
        rm -f $rep
        echo "ncu $c ok"
    fi
done
