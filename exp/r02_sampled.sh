#!/usr/bin/env bash
# Round 2 (session 2): sampled-block cost per entry vs the full sweep, and
# time-to-gap, on huge and medium (full BASELINE sizes).
mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
python bench.py --config huge --cache $CACHE --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # fill the cache
python bench.py --config medium --cache $CACHE --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
CFGS=huge,medium FRACS=1,2,4,8 N=64 timeout 900 python exp/sampled_cost.py > gpurun_out/sampled_cost.jsonl 2> gpurun_out/sampled_cost.err; echo "cost rc=$?"
timeout 900 python bench.py --mode ttg --config huge --cache $CACHE > gpurun_out/ttg_huge.json 2> gpurun_out/ttg_huge.err; echo "ttg huge rc=$?"
timeout 600 python bench.py --mode ttg --config medium --cache $CACHE > gpurun_out/ttg_medium.json 2> gpurun_out/ttg_medium.err; echo "ttg medium rc=$?"
SHORT="python bench.py --config medium --steps 5 --warmup 3 --no-cpu-baseline --cache $CACHE"
$SHORT > gpurun_out/med_short.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_primal -s 40 -c 4 \
      -o gpurun_out/prof_med $SHORT > gpurun_out/ncu_med.log 2>&1; echo "ncu medium rc=$?"
