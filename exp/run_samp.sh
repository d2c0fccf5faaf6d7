mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "sampled or exec_modes or bundle or set_state" > gpurun_out/samp_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/samp_tests.log
