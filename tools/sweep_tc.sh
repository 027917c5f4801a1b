# tcgen05 MTTKRP knob sweep on one config
C=${1:-c2}
timeout 120 python tools/time_modes.py $C 2>&1 | tail -1
for t in 0.5 0.85 1.0; do NTF_TC_TAILCOST=$t timeout 120 python tools/time_modes.py $C 2>&1 | tail -1 | sed "s/^/tail$t /"; done
for g in 1 2; do NTF_TC_TAILCOST=0.85 NTF_TC_G=$g timeout 120 python tools/time_modes.py $C 2>&1 | tail -1 | sed "s/^/G$g /"; done
for x in 3 4; do NTF_TC_TAILCOST=0.85 NTF_TC_XSTAGES=$x timeout 120 python tools/time_modes.py $C 2>&1 | tail -1 | sed "s/^/X$x /"; done
for d in 1 2 4 6 16 23; do NTF_TC_TAILCOST=0.85 NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1; done
