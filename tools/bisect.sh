run() { echo "== $C $*"; env "$@" timeout 60 python tools/time_modes.py $C 2>&1 | tail -1 | cut -c1-110; }
C=c3; run NTF_TC_DEBUG=0
C="custom auto 400 400 400 64 2"; run NTF_TC_DEBUG=0
C="custom auto 1000 1000 1000 80 1"; run NTF_TC_DEBUG=0
