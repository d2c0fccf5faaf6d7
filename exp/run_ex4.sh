mkdir -p gpurun_out
python bench.py --config multi --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
(echo "== multi"; CFG=multi N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_ex0.so exp/lib_exA.so exp/lib_exD.so exp/lib_ex0.so exp/lib_exD.so) > gpurun_out/ex4.log 2>&1
for L in exp/lib_ex0.so exp/lib_exA.so exp/lib_exD.so; do SPFOM_LIB=$PWD/$L python bench.py --config multi --steps 1000 --warmup 20 --cache /tmp/spfom_cache --no-cpu-baseline | tail -1; done > gpurun_out/ex4_multi.log 2>&1
