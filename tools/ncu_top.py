"""Summarise an ncu report: per kernel key metrics + top stall source lines."""
import csv, io, subprocess, sys
rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
idx = {k: h.index(k) for k in keys if k in h}
for r in rows[2:]:
    print({k: r[i][:60] for k, i in idx.items()})
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = src.split('"Kernel Name"')
for b in blocks[1:]:
    lines = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = lines[0][1][:80]
    hh = lines[1]
    ix = {n: i for i, n in enumerate(hh)}
    data = lines[2:]
    col = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[ix[col]] or 0) for r in data if len(r) > ix[col])
    print("==", name, "samples", tot)
    for r in sorted(data, key=lambda r: -float(r[ix[col]] or 0) if len(r) > ix[col] else 0)[:ntop]:
        print("  ", r[ix["Address"]][-5:], r[ix[col]], r[ix["Source"]][:80])
