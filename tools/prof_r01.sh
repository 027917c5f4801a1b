# launch list + full ncu captures of the top kernels of one bench step (c2)
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_short.json 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_tc_kernel -s 60 -c 1 -o gpurun_out/prof_mttkrp $B > gpurun_out/ncu_m.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_update -s 60 -c 1 -o gpurun_out/prof_update $B > gpurun_out/ncu_u.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:w_slice_kernel -s 60 -c 1 -o gpurun_out/prof_slice $B > gpurun_out/ncu_s.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ridge_factor_kernel -s 60 -c 1 -o gpurun_out/prof_ridge $B > gpurun_out/ncu_r.log 2>&1
