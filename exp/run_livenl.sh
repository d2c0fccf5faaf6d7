#!/bin/bash
# live-entry projection (SPFOM_LIVE_NL) + rows sorted by length in a bin: parity on the
# ragged / entry-mapped / medium paths, then K1 of base vs new on medium and huge
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "ragged or entry_mapped or sampled_stream or converge_preset or exec_modes or degenerate" > gpurun_out/livenl_tests.log 2>&1
echo "parity rc=$?" >> gpurun_out/livenl_tests.log
CFG=medium N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so paper_2602_22421_b200/libspfom.so exp/lib_base.so paper_2602_22421_b200/libspfom.so > gpurun_out/livenl_k1.log 2>&1
N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_base.so paper_2602_22421_b200/libspfom.so >> gpurun_out/livenl_k1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "medium" > gpurun_out/livenl_full.log 2>&1
echo "full rc=$?" >> gpurun_out/livenl_full.log
