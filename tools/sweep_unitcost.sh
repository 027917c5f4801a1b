# partition cost model sweep (diagnostic build): per-unit fixed share, in blocks
L=paper_1409_2383_b200/var_diag.so
for c in c5 c3 c2; do
  for u in 1 2.5 4 5.5; do
    echo "== $c unitcost $u $(NTF_VARIANT_LIB=$L NTF_TC_UNITCOST=$u timeout 300 python tools/time_modes.py $c 2>&1 | tail -1 | cut -c1-110)"
  done
done
