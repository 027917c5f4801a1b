"""Summarise an ncu launch-list CSV: per kernel count / mean duration / DRAM bytes."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {n: i for i, n in enumerate(h)}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[ix["Kernel Name"]][:70]][r[ix["Metric Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")))
tot = sum(sum(m.get("gpu__time_duration.sum", [0])) for m in agg.values())
for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
    t = m.get("gpu__time_duration.sum", [0])
    rd = m.get("dram__bytes_read.sum", [0])
    print(f"{k:70s} n={len(t):4d} mean_us={sum(t)/len(t)/1e3:8.2f} share={sum(t)/tot:6.1%} dram_rd_MB={sum(rd)/len(rd)/1e6:8.2f}")
