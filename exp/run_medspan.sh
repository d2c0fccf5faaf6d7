#!/bin/bash
# medium: per-bin K1 timeline (span build) at iterations 20 and 1500, ncu launch list of one step
mkdir -p gpurun_out
for it in 20 1500; do echo "== span IT=$it"; SPFOM_LIB=exp/lib_span.so CFG=medium IT=$it timeout 300 python exp/span_bins.py; done > gpurun_out/medspan.log 2>&1
timeout 300 python bench.py --config medium --steps 20 --warmup 5 > gpurun_out/med_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/med_launches.csv python bench.py --config medium --steps 2 --warmup 3 > gpurun_out/med_ncu.log 2>&1
echo done
