for C in c2 c3; do
for d in 22 534 16 528 0 512; do NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1; done
done
bash tools/tc_waits.sh c3 54 566
