mkdir -p gpurun_out
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python bench.py --config medium --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in huge medium; do echo "== $c"; CFG=$c N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_ex0.so exp/lib_ex4.so exp/lib_ex5.so exp/lib_ex8.so exp/lib_ex0.so exp/lib_ex5.so; done > gpurun_out/ex.log 2>&1
python bench.py --steps 20 --warmup 5 --cache /tmp/spfom_cache --no-cpu-baseline > gpurun_out/bench_ex.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/ex_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ex_tests.log
