#!/bin/bash
# medium K1: base (HEAD) vs sort-only vs 3-copy live entries without / with the sort vs runtime-bound single copy
mkdir -p gpurun_out
CFG=medium N=100 LATE=1500 timeout 1200 python exp/k1var.py exp/lib_base.so exp/lib_nl0.so exp/lib_nosort.so exp/lib_cur.so exp/lib_nl2.so exp/lib_base.so exp/lib_nl2.so > gpurun_out/livenl2_k1.log 2>&1
