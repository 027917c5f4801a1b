# Round-2 evidence run: GPU tests, bench lines, ncu launch list and full captures
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_gpu_tests.log 2>&1; tail -4 gpurun_out/r02_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02_bench_c5.log 2>&1; tail -c 600 gpurun_out/r02_bench_c5.log
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02_bench_$c.log 2>&1; tail -c 300 gpurun_out/r02_bench_$c.log; done
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
ls gpurun_out | head -50
