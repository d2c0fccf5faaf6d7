#!/bin/bash
# ncu --set full of the dominant K1 launch of medium (16-lane bin) and multi (k_primal_mp), each after a clean run
mkdir -p gpurun_out
for c in ${CFGS:-medium multi}; do
  CMD="python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --kernel-iters 3"
  $CMD > gpurun_out/prof_$c.log 2>&1 || { echo "$c run failed"; continue; }
  if [ $c = medium ]; then K='regex:k_primal_stream<.int.16,'; S=3; else K='regex:k_primal_mp'; S=3; fi
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -s $S -c 1 \
      -o gpurun_out/prof_$c $CMD > gpurun_out/ncu_$c.log 2>&1; echo "$c ncu rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$c.csv $CMD > /dev/null 2>&1
done
