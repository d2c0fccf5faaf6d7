#!/usr/bin/env bash
# round 2, fourth session: chunks of 3 rounds vs 2 (the product build), repeated processes, huge / medium
mkdir -p gpurun_out
P=paper_2602_22421_b200/libspfom.so; C=exp/lib_ch3.so
python exp/k1var.py $P $C $P $C $P $C > gpurun_out/v6_huge.txt 2>&1
CFG=medium python exp/k1var.py $P $C $P $C > gpurun_out/v6_medium.txt 2>&1
cat gpurun_out/v6_*.txt
