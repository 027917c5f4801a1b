# ms per outer iteration (graph replay) with CTA pairs vs single CTAs (diagnostic build)
L=paper_1409_2383_b200/var_diag.so
for c in c2 c3 c4 c5; do
  for cg in 1 2; do
    NTF_VARIANT_LIB=$L NTF_TC_CG=$cg timeout 300 python tools/step_time.py $c 10 2>&1 | tail -1
  done
done
