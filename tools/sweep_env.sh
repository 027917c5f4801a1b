#!/bin/bash
# c2 outer it/s under tuning env overrides: tools/sweep_env.sh "VAR=v ..." ...
for cfg in "" "$@"; do
  v=$(env $cfg timeout 200 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["frac"],4))')
  echo "== [$cfg] $v"
done
