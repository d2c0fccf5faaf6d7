#!/usr/bin/env bash
# round 2, fourth session: one-select piece masks, lazily formed Newton tolerance, chunk sizes 3 / 4 vs the product build
mkdir -p gpurun_out
L="paper_2602_22421_b200/libspfom.so exp/lib_hsel.so exp/lib_ltol.so exp/lib_ltol_hsel.so exp/lib_ch3.so exp/lib_ch4.so paper_2602_22421_b200/libspfom.so"
python exp/k1var.py $L > gpurun_out/v5_huge.txt 2>&1
CFG=medium python exp/k1var.py paper_2602_22421_b200/libspfom.so exp/lib_hsel.so exp/lib_ltol.so exp/lib_ltol_hsel.so > gpurun_out/v5_medium.txt 2>&1
CFG=multi LATE=600 python exp/k1var.py paper_2602_22421_b200/libspfom.so exp/lib_hsel.so exp/lib_ltol.so exp/lib_ltol_hsel.so > gpurun_out/v5_multi.txt 2>&1
cat gpurun_out/v5_*.txt
