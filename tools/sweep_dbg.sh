# tcgen05 MTTKRP bound analysis: per-mode times with diagnostic skip masks
# (2 skip MMA, 4 skip TMEM drain / epilogue math, 16 skip X loads)
L=paper_1409_2383_b200/var_diag.so
for c in ${CFGS:-c5 c3}; do
  for d in 0 2 4 16 6 20 18; do
    echo "== $c dbg $d $(NTF_VARIANT_LIB=$L NTF_TC_SLOTKS=${KS:-4} NTF_TC_DEBUG=$d timeout 300 python tools/time_modes.py $c 2>&1 | tail -1 | cut -c1-120)"
  done
done
