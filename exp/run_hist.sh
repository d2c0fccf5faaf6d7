mkdir -p gpurun_out
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python bench.py --config medium --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in huge medium; do echo "== $c"; CFG=$c N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so exp/lib_g2048.so exp/lib_h160.so exp/lib_h192.so exp/lib_h224.so exp/lib_base.so; done > gpurun_out/hist.log 2>&1
SPFOM_LIB=$PWD/exp/lib_sw.so CFGS=medium FRACS=2,8 N=64 timeout 900 python exp/sampled_cost.py > gpurun_out/sw_samp.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sampled or exec_modes or every or bundle" > gpurun_out/sw_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sw_tests.log
