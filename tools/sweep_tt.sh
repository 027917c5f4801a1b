for g in 2 4; do for d in 278 272 256; do echo "G=$g d=$d"; NTF_TC_G=$g NTF_TC_DEBUG=$d timeout 120 python tools/tc_times.py c2 12 2>&1 | tail -2; done; done
