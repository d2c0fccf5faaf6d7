mkdir -p gpurun_out
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python bench.py --config medium --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in huge medium; do echo "== $c"; CFG=$c N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so exp/lib_w8h256.so exp/lib_w12h256.so exp/lib_w12h256co0.so; done > gpurun_out/w12.log 2>&1
