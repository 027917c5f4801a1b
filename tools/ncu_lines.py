"""Per-CUDA-source-line warp-stall samples of an ncu report (cuda,sass view),
with the top stall reasons of each line."""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
                     + (["-k", kfilter] if kfilter else []),
                     capture_output=True, text=True).stdout
agg = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
fname = "?"
src = {}
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name":
        continue
    if hdr and len(r) > 4 and r[0].isdigit():
        try:
            v = float(r[4] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        agg[key] += v
        src[key] = r[1]
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try:
                    reasons[key][h[6:]] += float(r[i] or 0)
                except ValueError:
                    pass
tot = sum(agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:ntop]:
    top = sorted(reasons[k].items(), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{n}:{c:.0f}" for n, c in top if c > 0)
    print(f"{v:7.0f} {100*v/tot:5.1f}% {k[0]}:{k[1]}  {src[k][:70]}  [{rs}]")
