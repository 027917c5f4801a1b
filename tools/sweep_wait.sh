for C in c2 c3; do
for d in 22 1046 2070 3094 16 1040 2064 3088 0 1024 2048 3072; do NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1; done
done
