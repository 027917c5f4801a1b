# MTTKRP time per mode under NTF_TC_DEBUG skip masks (profiling only)
for C in "$@"; do
for d in 0 16 2 4 6 18 20 22 128; do
NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1
done
done
