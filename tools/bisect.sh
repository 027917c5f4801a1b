run() { echo "== $C $*"; env "$@" timeout 60 python tools/time_modes.py $C 2>&1 | tail -1 | cut -c1-110; }
for C in c2 c3 c4 "custom auto 1000 1000 1000 100 1" "custom auto 400 400 400 128 1"; do run NTF_TC_DEBUG=0; done
