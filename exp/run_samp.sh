mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "sampled or exec_modes or bundle or set_state" > gpurun_out/samp_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/samp_tests.log
for lib in paper_2602_22421_b200/libspfom.so exp/lib_nog4.so; do
  SPFOM_LIB=$lib FRACS=1,8,2 CFGS=huge timeout 900 python exp/sampled_cost.py
done > gpurun_out/samp_cost3.log 2>&1
