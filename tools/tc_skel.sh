export NTF_TC_TAILCOST=1.0
for d in 0 128 23 151; do NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py c2 2>&1 | tail -1; done
