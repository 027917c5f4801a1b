#!/bin/bash
# tools/var_debug.sh CFG var1 var2 ...: per-mode MTTKRP times under the debug skip masks
C=$1; shift
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_1409_2383_b200/var_$v.so; fi
  for d in ${DBGS:-0 16 2 4 6}; do
    echo "== $v dbg $d $(NTF_B200_LIB=$L NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1 | cut -c1-150)"
  done
done
