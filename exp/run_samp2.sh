mkdir -p gpurun_out
for lib in paper_2602_22421_b200/libspfom.so exp/lib_bulk.so; do
  SPFOM_LIB=$lib FRACS=8,4,2 timeout 900 python exp/sampled_cost.py
done > gpurun_out/samp_cost2.log 2>&1
