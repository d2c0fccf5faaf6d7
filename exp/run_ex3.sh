mkdir -p gpurun_out
for c in huge multi small; do python bench.py --config $c --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; done
for c in huge multi; do echo "== $c"; CFG=$c N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_ex0.so exp/lib_exA.so exp/lib_exB.so exp/lib_exC.so exp/lib_ex0.so exp/lib_exA.so exp/lib_exB.so; done > gpurun_out/ex3.log 2>&1
for L in exp/lib_ex0.so exp/lib_exA.so; do SPFOM_LIB=$PWD/$L python bench.py --config small --steps 1000 --warmup 20 --cache /tmp/spfom_cache --no-cpu-baseline | tail -1; done > gpurun_out/ex3_small.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "small or exec_modes or checkpoint or degenerate or converge_preset" > gpurun_out/ex3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ex3_tests.log
