#!/usr/bin/env bash
# round 2, fourth session: medium K1 against the SM shares of its four concurrent bin launches
# (-DSPFOM_DIAG_BIN_SMS library; SPFOM_BIN_SMS = shares of the active bins in bin order)
mkdir -p gpurun_out
export CFG=medium SHOW_BINS=1
for v in "" 3,6,29,110 3,7,30,108 3,6,30,109 3,7,29,109 4,7,30,107 3,7,31,107 3,8,30,107; do
  echo "== SPFOM_BIN_SMS=$v"
  if [ -z "$v" ]; then python exp/k1var.py exp/lib_sms.so; else SPFOM_BIN_SMS=$v python exp/k1var.py exp/lib_sms.so; fi
done > gpurun_out/shares_medium.txt 2>&1
cat gpurun_out/shares_medium.txt
