timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests8.log 2>&1; tail -12 gpurun_out/gpu_tests8.log
timeout 600 python -m pytest tests/test_fp32_parity.py -q -rA -k "c5" 2>&1 | grep -E "fp32 |passed|failed|Error|error" | head
timeout 600 python tools/mttkrp_error.py c4 10 2>&1 | tail -4
timeout 600 python tools/mttkrp_error.py c4 40 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_c5_t8.log 2> gpurun_out/bench_c5_t8.err; tail -c 2500 gpurun_out/bench_c5_t8.log; tail -3 gpurun_out/bench_c5_t8.err
