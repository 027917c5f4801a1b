run() { echo "== $*"; env "$@" timeout 60 python tools/time_modes.py $C 2>&1 | tail -1 | cut -c1-150; }
for C in c2 c3 c4; do run NTF_TC_DEBUG=0; run NTF_TC_DEBUG=6; run NTF_TC_DEBUG=16; done
C="custom auto 300 300 300 20 2"; run NTF_TC_DEBUG=0
C="custom auto 400 400 400 100 2"; run NTF_TC_DEBUG=0
C="custom auto 400 400 400 40 2"; run NTF_TC_DEBUG=0
