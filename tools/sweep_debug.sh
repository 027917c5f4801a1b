# per-role cost of the tcgen05 MTTKRP: time with roles disabled (NTF_TC_DEBUG bits)
C=${1:-c2}
for d in 0 1 2 4 8 16 6 7 31; do
  NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C 2>&1 | tail -1
done
