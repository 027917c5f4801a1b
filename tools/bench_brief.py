"""Key fields of the JSON line(s) in bench.py log files: python tools/bench_brief.py LOG..."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        r, e, c = d.get("roofline") or {}, d.get("e2e") or {}, d.get("clocks") or {}
        print(f"{path}: {d.get('value'):.4g} {d.get('unit')} ({d.get('ms_per_step'):.4g} ms/step)"
              f" frac {r.get('frac', 0):.3f} per-mode ms {[round(t, 4) for t in r.get('per_mode_ms', [])]}"
              f" share {r.get('mttkrp_share_of_step', 0):.2f} row-update {r.get('row_update_ms_mean', 0):.4f} ms"
              f" e2e {e.get('value', 0):.4g} rfe {e.get('final_rfe')} sm {c.get('sm_mhz')} {c.get('reasons')}")
