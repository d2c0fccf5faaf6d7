#!/bin/bash
# K1 setup/epilogue variants: shard proxy + span + k1var (huge, medium)
mkdir -p gpurun_out
for v in old new nosf nofs ch1; do
  lib=exp/lib_$v.so; [ $v = new ] && lib=paper_2602_22421_b200/libspfom.so
  echo "== $v"; SPFOM_LIB=$lib PS=1,8 timeout 600 python exp/shard_proxy.py 2>&1 | grep -v "^{"
done
for v in spanold span; do echo "== $v"; SPFOM_LIB=exp/lib_$v.so PS=1,8 timeout 300 python exp/span.py; done
N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_old.so paper_2602_22421_b200/libspfom.so exp/lib_ch1.so
CFG=medium N=100 LATE=1500 timeout 900 python exp/k1var.py exp/lib_old.so paper_2602_22421_b200/libspfom.so exp/lib_ch1.so
