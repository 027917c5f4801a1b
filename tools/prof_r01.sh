set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --no-kernel-timing --no-e2e --no-cpu-baseline > gpurun_out/bench_notiming.json 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_timing.json 2>&1
timeout 300 $B > gpurun_out/bench_short.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_tc_kernel -s 60 -c 1 -o gpurun_out/r01_mttkrp $B > gpurun_out/ncu_m.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_update_kernel -s 60 -c 1 -o gpurun_out/r01_update $B > gpurun_out/ncu_u.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ridge_factor_kernel -s 60 -c 1 -o gpurun_out/r01_ridge $B > gpurun_out/ncu_r.log 2>&1
ls -la gpurun_out
