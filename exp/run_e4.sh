mkdir -p gpurun_out
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
(echo "== huge"; CFG=huge N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so exp/lib_e4_1152.so exp/lib_h160.so paper_2602_22421_b200/libspfom.so exp/lib_e4_1408.so exp/lib_base.so paper_2602_22421_b200/libspfom.so) > gpurun_out/e4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/e4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/e4_tests.log
