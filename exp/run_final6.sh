#!/bin/bash
# round 2, fourth session: full gpu suite of the final tree with per-test durations, smoke, driver-window bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/final6_gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/final6_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final6_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/final6_bench.log 2>&1
