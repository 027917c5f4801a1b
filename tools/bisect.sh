for d in 0 16 22 6 18 20; do NTF_TC_DEBUG=$d timeout 60 python tools/time_modes.py c2 2>&1 | tail -1 | cut -c1-100; done
for d in 32 48; do NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py c2 > gpurun_out/w_$d.log 2>&1; done
