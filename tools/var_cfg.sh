#!/bin/bash
# tools/var_cfg.sh CFG STEPS var1 var2 ...: outer it/s of variant libraries on one config, twice each
C=$1; S=$2; shift 2
for rep in 1 2; do for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_1409_2383_b200/var_$v.so; fi
  echo "== $C $v $(NTF_B200_LIB=$L timeout 300 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), round(d["roofline"]["frac"],4))')"
done; done
