for s in 2 3 4 5 6; do echo "SX=$s"; NTF_TC_XSTAGES=$s NTF_TC_DEBUG=22 timeout 120 python tools/time_modes.py c2 2>&1 | tail -1; NTF_TC_XSTAGES=$s NTF_TC_DEBUG=16 timeout 120 python tools/time_modes.py c2 2>&1 | tail -1; done
for g in 1 2 4; do echo "G=$g"; NTF_TC_G=$g NTF_TC_DEBUG=22 timeout 120 python tools/time_modes.py c2 2>&1 | tail -1; done
