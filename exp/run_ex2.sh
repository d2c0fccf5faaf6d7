mkdir -p gpurun_out
for c in huge multi; do python bench.py --config $c --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "accuracy_gates" > gpurun_out/ex2_gates.log 2>&1; echo "gates rc=$?" >> gpurun_out/ex2_gates.log
for c in huge multi; do echo "== $c"; CFG=$c N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_ex0.so exp/lib_ex5p.so exp/lib_ex0.so exp/lib_ex5p.so; done > gpurun_out/ex2.log 2>&1
python bench.py --steps 20 --warmup 5 --cache /tmp/spfom_cache --no-cpu-baseline > gpurun_out/bench_ex2.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/ex2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ex2_tests.log
