import json, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
line = [l for l in sys.stdin.read().strip().splitlines() if l.startswith("{")][-1]
d = json.loads(line)
r = d.get("roofline", {})
print(tag, "value", round(d["value"], 2), "mttkrp_ms", [round(v, 4) for v in r.get("per_mode_ms", [])],
      "GB/s", [round(v) for v in r.get("per_mode_gbs", [])], "upd_ms", round(r.get("row_update_ms_mean", 0), 4),
      "frac", round(r.get("frac", 0), 3))
