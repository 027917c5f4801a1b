# per-role wait cycles of the tcgen05 MTTKRP (first and last CTA of every launch)
C=${1:-c2}
shift
mkdir -p gpurun_out
for d in "$@"; do
NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $C > gpurun_out/tcw_${C}_${d}.log 2>&1
done
