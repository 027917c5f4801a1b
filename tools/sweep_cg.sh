# tcgen05 MTTKRP: CTA pairs vs single CTAs (diagnostic build), per config
L=paper_1409_2383_b200/var_diag.so
for c in c2 c3 c4 c5; do
  for cg in 1 2; do
    echo "== $c cg $cg $(NTF_VARIANT_LIB=$L NTF_TC_CG=$cg timeout 300 python tools/time_modes.py $c 2>&1 | tail -1 | cut -c1-120)"
  done
done
for d in 2 4 16 6 20 18; do
  echo "== c5 cg 2 dbg $d $(NTF_VARIANT_LIB=$L NTF_TC_DEBUG=$d timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
done
echo "== c5 cg2 waits"; NTF_VARIANT_LIB=$L NTF_TC_DEBUG=32 timeout 300 python tools/time_modes.py c5 2>&1 | grep "tc cta" | head -12
