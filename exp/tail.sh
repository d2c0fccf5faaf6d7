#!/usr/bin/env bash
# ncu launch list of a short huge run: per-launch durations of K1, k_dual and friends
mkdir -p gpurun_out
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --cache /tmp/spfom_cache --config ${CFG:-huge}"
$CMD > gpurun_out/tail_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/tail_launches.csv $CMD > gpurun_out/tail_ncu.log 2>&1
echo "rc=$?"
