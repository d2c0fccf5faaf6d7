mkdir -p gpurun_out
for pr in converge paper; do for f in 1 8 2; do
  echo "== $pr FRAC=$f"; SPFOM_LIB=exp/lib_phg4.so PRESET=$pr FRAC=$f ITERS=40 timeout 600 python exp/phase.py
done; done > gpurun_out/samp_phase.log 2>&1
for f in 8 2; do echo "== span FRAC=$f"; SPFOM_LIB=exp/lib_spang4.so FRAC=$f PS=1 timeout 300 python exp/span.py; done >> gpurun_out/samp_phase.log 2>&1
