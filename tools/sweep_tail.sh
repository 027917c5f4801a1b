for t in 0.3 0.5 0.7 0.85 1.0; do NTF_TC_TAILCOST=$t timeout 120 python tools/time_modes.py ${1:-c2} 2>&1 | tail -1 | sed "s/^/tail$t /"; done
for x in 4 5 6; do NTF_TC_XSTAGES=$x timeout 120 python tools/time_modes.py ${1:-c2} 2>&1 | tail -1 | sed "s/^/X$x /"; done
