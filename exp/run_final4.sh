#!/bin/bash
# round 2, fourth session (re-created container, rebuilt libraries): full gpu suite, smoke, driver-window bench, other configs
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final4_gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/final4_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final4_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/final4_bench.log 2>&1
for c in medium multi small; do timeout 900 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline >> gpurun_out/final4_other.log 2>&1; done
