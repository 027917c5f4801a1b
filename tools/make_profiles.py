"""Write the round's ncu summaries into profiles/ from gpurun_out/ reports.

  python tools/make_profiles.py r01

Inputs (produced by tools/prof_r01.sh on the GPU box): gpurun_out/launches.csv
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
launch list of `bench.py --steps 3 --warmup 3`), gpurun_out/prof_*.ncu-rep
(--set full captures of single launches).  Outputs: profiles/<tag>_launches.txt,
profiles/<tag>_<kernel>_ncu.txt, profiles/ncu_traffic.json.
"""
import collections, csv, io, json, os, subprocess, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.path.join(REPO, "profiles")
os.makedirs(out_dir, exist_ok=True)
gro = os.path.join(REPO, "gpurun_out")


def launches():
    rows = [r for r in csv.reader(open(os.path.join(gro, "launches.csv"))) if len(r) > 10]
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        v = float(r[ix["Metric Value"]].replace(",", ""))
        agg[r[ix["Kernel Name"]]][r[ix["Metric Name"]]].append(v)
    tot = sum(sum(m.get("gpu__time_duration.sum", [0])) for m in agg.values())
    lines = [f"# ncu launch list of `python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline` (c2)",
             "# --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
             "# per-launch times are cold-cache and serialised: compare SHARES with bench.py, not absolutes",
             f"{'kernel':80s} {'n':>5s} {'mean_us':>9s} {'share':>7s} {'dram_rd_MB':>11s} {'dram_wr_MB':>11s}"]
    traffic = {}
    for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
        t = m.get("gpu__time_duration.sum", [0.0])
        rd = m.get("dram__bytes_read.sum", [0.0])
        wr = m.get("dram__bytes_write.sum", [0.0])
        lines.append(f"{k[:80]:80s} {len(t):5d} {sum(t)/len(t)/1e3:9.2f} {sum(t)/tot:7.1%} "
                     f"{sum(rd)/len(rd)/1e6:11.2f} {sum(wr)/len(wr)/1e6:11.2f}")
        if "mttkrp" in k and "reduce" not in k:
            traffic[k] = (sum(rd) + sum(wr)) / len(rd)
    with open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if traffic:
        top = max(traffic.items(), key=lambda kv: kv[1])
        with open(os.path.join(out_dir, "ncu_traffic.json"), "w") as fh:
            json.dump({"c2": top[1], "kernel": top[0], "source": f"profiles/{tag}_launches.txt",
                       "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (mean)"}, fh, indent=1)
    print("\n".join(lines))


def details(rep, name):
    path = os.path.join(gro, rep)
    if not os.path.exists(path):
        return
    d = subprocess.run(["ncu", "-i", path, "--page", "details"], capture_output=True, text=True).stdout
    keep = [ln for ln in d.splitlines() if ln.strip() and not set(ln.strip()) <= set("-")]
    src = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_lines.py"), path, "30"],
                         capture_output=True, text=True).stdout
    with open(os.path.join(out_dir, f"{tag}_{name}_ncu.txt"), "w") as fh:
        fh.write(f"# ncu --set full --import-source on --clock-control none, one launch ({rep})\n")
        fh.write("\n".join(keep[:400]) + "\n\n# warp-stall samples by CUDA source line (tools/ncu_lines.py)\n")
        fh.write(src)


launches()
for rep, name in [("prof_mttkrp.ncu-rep", "mttkrp_tc"), ("prof_update.ncu-rep", "row_update"),
                  ("prof_slice.ncu-rep", "w_slice"), ("prof_ridge.ncu-rep", "ridge")]:
    details(rep, name)
