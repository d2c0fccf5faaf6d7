#!/usr/bin/env bash
# E = 7 entries per lane on 8 lanes (huge rows in the G = 8 bin) at 8 / 12 / 16 warps per SM vs the product build
mkdir -p gpurun_out
python exp/k1var.py paper_2602_22421_b200/libspfom.so exp/lib_e7w12.so exp/lib_e7w8.so exp/lib_e7w16.so paper_2602_22421_b200/libspfom.so > gpurun_out/e7_huge.txt 2>&1
cat gpurun_out/e7_huge.txt
