# c2 step time: release (auto CTA grouping) vs diagnostic single / pair builds, same box
for r in 1 2; do
  timeout 300 python tools/step_time.py c2 20
  NTF_VARIANT_LIB=paper_1409_2383_b200/var_diag.so NTF_TC_CG=1 timeout 300 python tools/step_time.py c2 20
  NTF_VARIANT_LIB=paper_1409_2383_b200/var_diag.so NTF_TC_CG=2 timeout 300 python tools/step_time.py c2 20
done
timeout 300 python tools/time_modes.py c2
NTF_VARIANT_LIB=paper_1409_2383_b200/var_diag.so NTF_TC_CG=1 timeout 300 python tools/time_modes.py c2
