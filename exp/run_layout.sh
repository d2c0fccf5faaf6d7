mkdir -p gpurun_out
grep -o -m1 'avx2' /proc/cpuinfo > gpurun_out/layout.log; nproc >> gpurun_out/layout.log
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
SPFOM_TRACE_CREATE=1 python exp/e2e_phases.py >> gpurun_out/layout.log 2>&1
python bench.py --steps 20 --warmup 5 --cache /tmp/spfom_cache --no-cpu-baseline > gpurun_out/bench_layout.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/layout_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/layout_tests.log
