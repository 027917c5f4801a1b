timeout 900 python -m pytest tests -m gpu -x -q -k "tcgen05 or mttkrp or small_fits or c1 or interleaved" > gpurun_out/gpu_tests7.log 2>&1; tail -3 gpurun_out/gpu_tests7.log
timeout 300 bash tools/quick_modes.sh 2>&1
for v in diag epi16; do
  echo "== $v c5 $(NTF_VARIANT_LIB=paper_1409_2383_b200/var_$v.so timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
  echo "== $v c5 dbg18 $(NTF_VARIANT_LIB=paper_1409_2383_b200/var_$v.so NTF_TC_DEBUG=18 timeout 300 python tools/time_modes.py c5 2>&1 | tail -1 | cut -c1-120)"
done
timeout 1200 python -m pytest tests/test_fp32_parity.py -q -rA -k "config_final or fp64_engine or c5" 2>&1 | grep -E "fp32 |passed|failed|PASS|FAIL" | head -30
