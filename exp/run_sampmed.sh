# ncu launch lists of medium, converge preset, full sweep vs B = m/2 (per-bin K1 durations)
mkdir -p gpurun_out
python bench.py --config medium --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in 1 2 8; do
  FRAC=$f ITERS=8 python exp/samp_medium.py > gpurun_out/sampmed_$f.log 2>&1 && \
  FRAC=$f ITERS=8 timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv \
     --log-file gpurun_out/sampmed_launch_$f.csv python exp/samp_medium.py > /dev/null 2>&1; echo "frac $f rc=$?"
done
