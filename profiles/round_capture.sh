#!/bin/bash
# One round's measurement pass (run under gpurun on ONE B200, from the repo root):
# bench lines for every config (with the reference CPU baseline), the default bench and the
# reference arm, then an ncu launch list + one full-set capture per config.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/$TAG/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in cfg1 cfg2 cfg2b cfg3 cfg4; do
    timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err
    echo "bench $c rc=$?"
done
timeout 400 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err; echo "default rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/$TAG/bench_reference.json 2>&1; echo "reference rc=$?"
for a in "cfg1 k_general_sort" "cfg2 k_general_sort" "cfg2b k_general_sort" "cfg3 k_tile_sort" "cfg4 k_permute"; do
    set -- $a
    timeout 600 bash profiles/ncu_capture.sh $1 $TAG $2 && echo "ncu $1 ok"
done
