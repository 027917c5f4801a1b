# X-streaming skeleton (NTF_TC_DEBUG=6: no MMA, no drain) vs units size G, and commit latency
for C in c2 c3; do
for g in 1 2 4; do echo "G=$g"; NTF_TC_G=$g NTF_TC_DEBUG=6 timeout 120 python tools/time_modes.py $C 2>&1 | tail -1; done
for d in 22 86 0; do NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1; done
for g in 1 2 4; do echo "G=$g full"; NTF_TC_G=$g timeout 120 python tools/time_modes.py $C 2>&1 | tail -1; done
done
