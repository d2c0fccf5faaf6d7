mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
bash profiles/collect.sh > gpurun_out/collect.log 2>&1
CFGS=huge,medium FRACS=1,2,4,8 N=64 timeout 1200 python exp/sampled_cost.py > gpurun_out/sampled_cost2.jsonl 2> gpurun_out/sampled_cost2.err; echo "cost rc=$?"
