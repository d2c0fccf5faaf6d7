mkdir -p gpurun_out
CACHE=/tmp/spfom_cache
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_short.log 2>&1; echo "bench short rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
bash profiles/collect.sh > gpurun_out/collect.log 2>&1; cat gpurun_out/collect.log
WORKLOAD=huge bash exp/prof_late.sh > gpurun_out/late_rc.log 2>&1; cat gpurun_out/late_rc.log
for c in medium multi small; do python bench.py --config $c --steps 1000 --warmup 20 --cache $CACHE --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
