#!/bin/bash
# bench lines for every config (with the reference CPU baseline), the default line and the
# reference arm; run under gpurun from the repo root:  bash profiles/bench_all.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/$TAG/gpu.txt
for c in cfg1 cfg1sw cfg2 cfg2b cfg3 cfg3sw cfg4 cfg4s cfg5; do
    timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err
    echo "bench $c rc=$?"
done
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/$TAG/bench_reference.json 2>&1; echo "reference rc=$?"
