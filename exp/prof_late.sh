#!/usr/bin/env bash
# ncu --set full of one K1 launch late in the run (steady state, ~1500 iterations in)
mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
CMD="python bench.py --steps 1600 --warmup 3 --no-cpu-baseline --cache $CACHE"
$CMD > gpurun_out/late.log 2>&1; echo "late rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_primal_stream -s 1500 -c 1 \
    -o gpurun_out/prof_late $CMD > gpurun_out/ncu_late.log 2>&1; echo "ncu late rc=$?"
