#!/usr/bin/env bash
# ncu --set full of the K1 stream kernel on the huge config (one launch)
mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
SHORT="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --kernel-iters 3 --cache $CACHE"
$SHORT > gpurun_out/short.log 2>&1; echo "short rc=$?"; tail -1 gpurun_out/short.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:${1:-k_primal} -s 20 -c 1 \
    -o gpurun_out/prof_${2:-k1} $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
