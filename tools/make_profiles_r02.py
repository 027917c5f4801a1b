"""Write round-2 ncu summaries into profiles/ from gpurun_out/ (tools/prof_r02.sh).

  python tools/make_profiles_r02.py

Outputs: profiles/r02_launches_c2.txt (per-kernel launch list of two c2 bench
steps), profiles/r02_mttkrp_<cfg>_ncu.txt (--set full details of one mode-1
tcgen05 MTTKRP launch at c5, c3, c4) and profiles/ncu_traffic.json (DRAM
bytes read + written per MTTKRP launch, per config: the bench's
roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRO = os.path.join(REPO, "gpurun_out")
OUT = os.path.join(REPO, "profiles")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "s": 1.0}


def launch_list(name, title):
    rows = [r for r in csv.reader(open(os.path.join(GRO, name))) if len(r) > 10]
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1.0)
        agg[r[ix["Kernel Name"]]][r[ix["Metric Name"]]].append(v)
    tot = sum(sum(m.get("gpu__time_duration.sum", [0])) for m in agg.values())
    lines = [f"# {title}",
             "# --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
             "# per-launch times are cold-cache and serialised: compare SHARES with bench.py, not absolutes",
             f"{'kernel':80s} {'n':>5s} {'mean_us':>9s} {'share':>7s} {'dram_rd_MB':>11s} {'dram_wr_MB':>11s}"]
    traffic = None
    for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
        t = m.get("gpu__time_duration.sum", [0.0])
        rd = m.get("dram__bytes_read.sum", [0.0])
        wr = m.get("dram__bytes_write.sum", [0.0])
        lines.append(f"{k[:80]:80s} {len(t):5d} {sum(t) / len(t) * 1e6:9.2f} {sum(t) / tot:7.1%} "
                     f"{sum(rd) / len(rd) / 1e6:11.2f} {sum(wr) / len(wr) / 1e6:11.2f}")
        if "mttkrp_tc_kernel" in k:
            traffic = (k, sum(rd) / len(rd) + sum(wr) / len(wr))
    return lines, traffic


def full_capture(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    vals = {a: (b, c) for a, b, c in zip(h, u, v)}
    for a in list(vals):  # section-qualified names ("TPC.TriageCompute.sm__pipe_...") also under their metric name
        vals.setdefault(a.rsplit(".Triage", 1)[-1].split(".", 1)[-1] if ".Triage" in a else a, vals[a])
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout

    def num(k):
        unit, val = vals[k]
        return float(val.replace(",", "")) * UNIT.get(unit, 1.0)

    return vals, det, num


def main():
    os.makedirs(OUT, exist_ok=True)
    traffic = {"note": "dram__bytes_read.sum + dram__bytes_write.sum per tcgen05 MTTKRP launch (bytes)"}
    lines, tr = launch_list("r02_launches_c2.csv",
                            "ncu launch list of `python bench.py --config c2 --steps 2 --warmup 3 --no-e2e "
                            "--no-cpu-baseline` (round 2)")
    open(os.path.join(OUT, "r02_launches_c2.txt"), "w").write("\n".join(lines) + "\n")
    if tr:
        traffic["c2"] = {"bytes_per_launch": tr[1], "kernel": tr[0], "source": "profiles/r02_launches_c2.txt"}
    if os.path.exists(os.path.join(GRO, "r02_launches_c5.csv")):
        lines5, _ = launch_list("r02_launches_c5.csv",
                                "ncu launch list of `python bench.py --steps 2 --warmup 3 --no-e2e "
                                "--no-cpu-baseline` (c5, round 2, final tree)")
        open(os.path.join(OUT, "r02_launches_c5.txt"), "w").write("\n".join(lines5) + "\n")
    keep = ("Duration", "SM Frequency", "DRAM Frequency", "DRAM Throughput", "Memory Throughput",
            "Executed Ipc", "Issue Slots Busy", "Registers Per Thread", "Grid Size", "Block Size",
            "Cluster Size", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "L1/TEX Hit Rate",
            "L2 Hit Rate", "Mem Busy")
    for cfg in ("c5", "c3", "c4"):
        rep = os.path.join(GRO, f"r02_mttkrp_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        vals, det, num = full_capture(rep)
        name = vals.get("Kernel Name", ("", "?"))[1]
        rd, wr, dur = num("dram__bytes_read.sum"), num("dram__bytes_write.sum"), num("gpu__time_duration.sum")
        extra = []
        for k in ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                  "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                  "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                  "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
                  "smsp__inst_executed.sum"):
            if k in vals:
                extra.append(f"{k} = {vals[k][1]} {vals[k][0]}")
        out = [f"# ncu --set full --clock-control none --import-source on, one mode-1 launch "
               f"(`tools/prof_mttkrp.py --config {cfg} --modes 1 --iters 1`, -k regex:mttkrp_tc -s 2 -c 1)",
               f"kernel: {name}",
               f"dram bytes read {rd / 1e9:.4f} GB, written {wr / 1e6:.3f} MB, duration {dur * 1e3:.4f} ms, "
               f"DRAM throughput {(rd + wr) / dur / 1e12:.3f} TB/s"]
        out += extra
        out += [ln.rstrip() for ln in det.splitlines() if any(k in ln for k in keep)]
        open(os.path.join(OUT, f"r02_mttkrp_{cfg}_ncu.txt"), "w").write("\n".join(out) + "\n")
        traffic[cfg] = {"bytes_per_launch": rd + wr, "kernel": name,
                        "source": f"profiles/r02_mttkrp_{cfg}_ncu.txt"}
    # the fp64-arithmetic engine (DMMA pipeline) at 1000^3 fp64, R = 50, mode 1
    rep = os.path.join(GRO, "r02_mttkrp_cc64.ncu-rep")
    if os.path.exists(rep):
        vals, det, num = full_capture(rep)
        name = vals.get("Kernel Name", ("", "?"))[1]
        rd, wr, dur = num("dram__bytes_read.sum"), num("dram__bytes_write.sum"), num("gpu__time_duration.sum")
        flops = 2.0 * 1e9 * 56  # 7 issued 8-column blocks
        out = ["# ncu --set full --clock-control none --import-source on, one mode-1 launch of the fp64-arithmetic "
               "engine (`tools/time_modes.py custom cuda_core 1000 1000 1000 50 1 float64`, -k regex:mttkrp_cc -s 2 -c 1)",
               f"kernel: {name}",
               f"dram bytes read {rd / 1e9:.4f} GB, written {wr / 1e6:.3f} MB, duration {dur * 1e3:.4f} ms, "
               f"DRAM throughput {(rd + wr) / dur / 1e12:.3f} TB/s, issued DMMA flops {flops / dur / 1e12:.1f} TFLOP/s "
               "of 37.0 measured (tools/ubench/f64_rate.cu)"]
        for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_tensor_op_dmma.sum", "smsp__inst_executed.sum"):
            if k in vals:
                out.append(f"{k} = {vals[k][1]} {vals[k][0]}")
        out += [ln.rstrip() for ln in det.splitlines() if any(k in ln for k in keep)]
        open(os.path.join(OUT, "r02_mttkrp_cc64_ncu.txt"), "w").write("\n".join(out) + "\n")
    json.dump(traffic, open(os.path.join(OUT, "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
