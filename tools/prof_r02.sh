# Round-2 evidence run: GPU tests, bench lines, ncu launch list and full captures
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_gpu_tests.log 2>&1; tail -4 gpurun_out/r02_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02_bench_c5.log 2>&1; tail -c 600 gpurun_out/r02_bench_c5.log
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02_bench_$c.log 2>&1; tail -c 300 gpurun_out/r02_bench_$c.log; done
timeout 900 python bench.py --config c2 --steps 20 --warmup 5 --sharded --no-cpu-baseline > gpurun_out/r02_bench_c2_sharded.log 2>&1; tail -c 300 gpurun_out/r02_bench_c2_sharded.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_bench_reference_c5.log 2>&1; tail -c 400 gpurun_out/r02_bench_reference_c5.log
# launch list of two c2 bench steps (kernel shares)
B="python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/r02_c2_short.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_c2.csv $B > gpurun_out/r02_ncu_launch.log 2>&1
# full captures of the tcgen05 MTTKRP at c5, c3, c4 (mode 1)
for c in c5 c3 c4; do
  timeout 300 python tools/prof_mttkrp.py --config $c --modes 1 --iters 1 > gpurun_out/r02_prof_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:mttkrp_tc -s 2 -c 1 -o gpurun_out/r02_mttkrp_$c python tools/prof_mttkrp.py --config $c --modes 1 --iters 1 > gpurun_out/r02_ncu_$c.log 2>&1
done
# full capture of the fp64-arithmetic engine (DMMA pipeline) at 1000^3 fp64, R = 50
C="python tools/time_modes.py custom cuda_core 1000 1000 1000 50 1 float64"
timeout 300 $C > gpurun_out/r02_prof_cc64.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mttkrp_cc -s 2 -c 1 -f -o gpurun_out/r02_mttkrp_cc64 $C > gpurun_out/r02_ncu_cc64.log 2>&1
# the fp64 engine's per-mode times (DESIGN 4b) and the c1 bench line
for a in "1000 1000 1000 20 3 float64" "1000 1000 1000 50 3 float64" "1000 1000 1000 64 3 float64" "1000 1000 1000 100 3 float64" "400 400 400 20 5 float64" "5000 500 200 32 3 float64" "1000 1000 1000 50 3 float32" "400 400 400 150 3 float32"; do timeout 200 python tools/time_modes.py custom cuda_core $a | tail -1; done > gpurun_out/r02_fp64_engine_times.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/r02_bench_c1.log 2>&1; tail -c 300 gpurun_out/r02_bench_c1.log
timeout 120 ./tools/ubench/f64_rate > gpurun_out/r02_f64_rate.log 2>&1
ls gpurun_out | head -60
