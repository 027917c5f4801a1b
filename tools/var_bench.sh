#!/bin/bash
# A/B the variant libraries against the default on c2: tools/var_bench.sh var1 var2 ...
for rep in 1 2; do
  for v in default "$@"; do
    if [ $v = default ]; then L=""; else L=paper_1409_2383_b200/var_$v.so; fi
    echo "== $v $(NTF_B200_LIB=$L timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"])')"
  done
done
