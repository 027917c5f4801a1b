timeout 900 python -m pytest tests -m gpu -x -q -k "tcgen05 or mttkrp or sharded_tensor or peer" > gpurun_out/gpu_tests9.log 2>&1; tail -3 gpurun_out/gpu_tests9.log
timeout 600 python tools/mttkrp_error.py c4 40 2>&1 | tail -3
timeout 900 python -m pytest tests/test_fp32_parity.py -q -rA -k "config_final" 2>&1 | grep -E "^fp32 |passed|failed" | head -12
bash tools/sweep_c5.sh
timeout 300 python tools/time_modes.py custom cuda_core 1000 1000 1000 50 2 float64 2>&1 | tail -1
timeout 300 python tools/time_modes.py custom cuda_core 400 400 400 20 2 float64 2>&1 | tail -1
