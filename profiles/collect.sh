#!/usr/bin/env bash
# Reproduce the round's measurements on a B200 (run from the repo root under gpurun):
#   1. the bench line (default arguments)             -> gpurun_out/bench.log
#   2. ncu launch list of the same bench command      -> gpurun_out/launches.csv
#   3. one `ncu --set full` capture of K1 (k_primal)  -> gpurun_out/prof_k1.ncu-rep
# Each ncu step runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
python bench.py --cache $CACHE > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
SHORT="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --kernel-iters 3 --cache $CACHE"
$SHORT > gpurun_out/short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
$SHORT > gpurun_out/short2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_primal -s 4 -c 1 \
      -o gpurun_out/prof_k1 $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
