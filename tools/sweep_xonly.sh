# X-streaming only (MMA + drain skipped): tail weighting and ring depth
for t in 0.3 0.5 1.0; do NTF_TC_DEBUG=6 NTF_TC_TAILCOST=$t timeout 120 python tools/time_modes.py c2 2>&1 | tail -1 | sed "s/^/tail$t /"; done
for x in 2 3 4 6; do NTF_TC_DEBUG=6 NTF_TC_XSTAGES=$x timeout 120 python tools/time_modes.py c2 2>&1 | tail -1 | sed "s/^/X$x /"; done
for x in 2 3; do NTF_TC_XSTAGES=$x timeout 120 python tools/time_modes.py c2 2>&1 | tail -1 | sed "s/^/full X$x /"; done
