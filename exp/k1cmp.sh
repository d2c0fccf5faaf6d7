#!/usr/bin/env bash
# Compare K1 variants: SPFOM_LIB=<so> bench.py (short), print it/s and K1 ms.
mkdir -p gpurun_out
for so in paper_2602_22421_b200/libspfom.so "$@"; do
  SPFOM_LIB=$PWD/$so python bench.py --steps 300 --warmup 10 --no-cpu-baseline --kernel-iters 30 --cache /tmp/spfom_cache > gpurun_out/k1cmp_$(basename $so).log 2>&1
  tail -1 gpurun_out/k1cmp_$(basename $so).log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', round(d['value'],1), 'it/s  K1 ms', round(d['roofline']['k1_ms_avg'],4), 'frac', round(d['roofline']['frac'],3), 'passes', d.get('newton_passes_per_segment_iteration'))" || tail -5 gpurun_out/k1cmp_$(basename $so).log
done
