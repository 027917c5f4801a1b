set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/c5_clocks.csv &
SMI=$!
python tools/prof_mttkrp.py --config c5 --modes 123 --iters 5 > gpurun_out/c5_plain.log 2>&1
kill $SMI
python tools/prof_mttkrp.py --config c5 --modes 1 --iters 1 > gpurun_out/c5_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mttkrp_tc -s 2 -c 1 -o gpurun_out/c5_mode1 python tools/prof_mttkrp.py --config c5 --modes 1 --iters 1 > gpurun_out/c5_ncu.log 2>&1
echo done
