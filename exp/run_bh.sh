mkdir -p gpurun_out
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python bench.py --config medium --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in huge medium; do echo "== $c"; CFG=$c N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so exp/lib_bh512.so exp/lib_bh1024.so exp/lib_bh2048.so exp/lib_base.so exp/lib_bh1024.so; done > gpurun_out/bh.log 2>&1
SPFOM_LIB=$PWD/exp/lib_bh1024.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "entry_mapped or converge_preset_lockstep or paper_preset or ragged or theta or exec_modes or step_timed or nccl or averaging or residuals" > gpurun_out/bh_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/bh_tests.log
