# quick check: GPU parity tests of the MTTKRP + per-mode timings and CTA timelines
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "$@"; do
for d in 0 16 22 6; do NTF_TC_DEBUG=$d timeout 120 python tools/time_modes.py $c 2>&1 | tail -1; done
NTF_TC_DEBUG=256 timeout 120 python tools/tc_times.py $c 2>&1 | tail -3
done
