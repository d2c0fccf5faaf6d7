mkdir -p gpurun_out
python bench.py --config medium --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
(echo "== medium k1var"; CFG=medium N=100 LATE=1500 timeout 600 python exp/k1var.py exp/lib_head.so paper_2602_22421_b200/libspfom.so exp/lib_head.so paper_2602_22421_b200/libspfom.so) > gpurun_out/split.log 2>&1
for L in exp/lib_head.so paper_2602_22421_b200/libspfom.so exp/lib_sb0.so; do SPFOM_LIB=$PWD/$L CFGS=medium FRACS=1,2,8 N=64 timeout 600 python exp/sampled_cost.py; done > gpurun_out/split_samp.log 2>&1
for f in 1 2 8; do echo "== FRAC $f"; SPFOM_LIB=$PWD/exp/lib_ph.so CFG=medium FRAC=$f ITERS=40 timeout 300 python exp/phase.py; done > gpurun_out/split_phase.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ragged or medium or every or sampled_stream" > gpurun_out/split_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/split_tests.log
