mkdir -p gpurun_out
python bench.py --config huge --cache /tmp/spfom_cache --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
(echo "== huge"; CFG=huge N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so exp/lib_pre.so exp/lib_nopre.so exp/lib_pre.so exp/lib_base.so) > gpurun_out/pre.log 2>&1
SPFOM_LIB=$PWD/exp/lib_pre.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "entry_mapped or converge_preset_lockstep or paper_preset or ragged or theta or exec_modes or step_timed or nccl" > gpurun_out/pre_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pre_tests.log
