# c5 tcgen05 MTTKRP tuning sweep (diagnostic builds): epilogue load width, G, ring depth
for v in diag lw8; do
  L=paper_1409_2383_b200/var_$v.so
  echo "== $v c5 $(NTF_VARIANT_LIB=$L timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
  echo "== $v c5 dbg18 $(NTF_VARIANT_LIB=$L NTF_TC_DEBUG=18 timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
done
L=paper_1409_2383_b200/var_diag.so
for g in 3 5; do
  echo "== G=$g c5 $(NTF_VARIANT_LIB=$L NTF_TC_G=$g timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
done
echo "== G=5 lw8 c5 $(NTF_VARIANT_LIB=paper_1409_2383_b200/var_lw8.so NTF_TC_G=5 timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
