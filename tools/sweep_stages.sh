# MTTKRP ring-depth sweep (c2): X / factor-row / W stages
for cfg in "4 3 3" "5 2 2" "5 3 2" "6 2 2" "5 2 3"; do
  set -- $cfg
  NTF_TC_XSTAGES=$1 NTF_TC_FSTAGES=$2 NTF_TC_WSTAGES=$3 timeout 120 python tools/time_modes.py c2 2>&1 | tail -1 | sed "s/^/x$1 f$2 w$3 /"
done
