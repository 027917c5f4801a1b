run() { echo "== $C $*"; env "$@" timeout 60 python tools/time_modes.py $C 2>&1 | tail -1 | cut -c1-110; }
C=c2; run NTF_TC_MINSTAGES=4; run NTF_TC_MINSTAGES=3
C=c3; run NTF_TC_MINSTAGES=4; run NTF_TC_MINSTAGES=3; run NTF_TC_G=4 NTF_TC_XSTAGES=3; run NTF_TC_G=2
C="custom auto 1000 1000 1000 100 1"; run NTF_TC_MINSTAGES=4; run NTF_TC_G=3 NTF_TC_XSTAGES=2; run NTF_TC_MINSTAGES=2
C=c4; run NTF_TC_MINSTAGES=4; run NTF_TC_MINSTAGES=3
