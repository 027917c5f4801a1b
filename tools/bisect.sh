run() { echo "== $C $*"; env "$@" timeout 60 python tools/time_modes.py $C 2>&1 | tail -1 | cut -c1-110; }
for uc in 6 8 12; do
for C in c2 c3 c4 "custom auto 400 400 400 100 2" "custom auto 1000 1000 1000 100 1" "custom auto 400 400 400 64 2"; do run NTF_TC_UNITCOST=$uc; done
done
