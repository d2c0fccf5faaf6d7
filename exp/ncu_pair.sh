#!/usr/bin/env bash
# ncu (memory / scheduler sections) of one early K1 launch for each library given
mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
SHORT="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --kernel-iters 3 --cache $CACHE"
for lib in "$@"; do
  name=$(basename $lib .so)
  SPFOM_LIB=$PWD/$lib $SHORT > gpurun_out/short_$name.log 2>&1 || { echo "plain run of $name failed"; continue; }
  SPFOM_LIB=$PWD/$lib ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Chart \
     --section SchedulerStats --section WarpStateStats --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy \
     --metrics lts__t_sectors_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,lts__t_sector_hit_rate.ratio,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum,lts__t_requests_srcunit_tex_op_red_lookup_miss.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex.sum,lts__d_sectors.sum,sm__inst_executed_pipe_lsu.sum,smsp__inst_executed_op_global_red.sum \
     --clock-control none -k regex:k_primal_stream -s 10 -c 1 -o gpurun_out/ncu_$name $SHORT > gpurun_out/ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
done
