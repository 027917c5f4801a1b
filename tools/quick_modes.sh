# per-mode MTTKRP + row-update times of every BASELINE fp32 config (tools/time_modes.py)
for c in c2 c3 c4 c5; do timeout 300 python tools/time_modes.py $c; done
