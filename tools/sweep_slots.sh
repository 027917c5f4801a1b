# X ring slot size / ring depth sweep of the tcgen05 MTTKRP (diagnostic build)
L=paper_1409_2383_b200/var_diag.so
for c in c2 c3 c4 c5; do
  for k in 1 2 4; do
    echo "== $c slot_ks $k $(NTF_VARIANT_LIB=$L NTF_TC_SLOTKS=$k timeout 300 python tools/time_modes.py $c 2>&1 | tail -1 | cut -c1-160)"
  done
done
for k in 1 4; do
  echo "== c5 waits slot_ks $k"; NTF_VARIANT_LIB=$L NTF_TC_SLOTKS=$k NTF_TC_DEBUG=32 timeout 300 python tools/time_modes.py c5 2>&1 | grep "tc cta" | head -12
done
