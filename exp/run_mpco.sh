#!/usr/bin/env bash
# round 2, fourth session: multi-period kernel with the CHECK-pass output (ids parked in shared memory) vs the product build
mkdir -p gpurun_out
P=paper_2602_22421_b200/libspfom.so; C=exp/lib_mpco.so
CFG=multi LATE=600 python exp/k1var.py $P $C $P $C > gpurun_out/mpco_multi.txt 2>&1
cat gpurun_out/mpco_multi.txt
SPFOM_LIB=$PWD/exp/lib_mpco.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -k "multi" -x > gpurun_out/mpco_tests.txt 2>&1; tail -3 gpurun_out/mpco_tests.txt
