#!/usr/bin/env python
"""Benchmark: NTF outer iterations/sec on B200 (BASELINE.json metric).

One *step* is one ADMoM outer iteration of the reference algorithm
(solver.iterate, reference solver.py:295-327): ``inner`` Gauss-Seidel sweeps
x 3 modes of (dense MTTKRP -> ridge Cholesky -> row solve), with the
projection / dual step / residuals / adaptation fused in.  Default workload:
BASELINE config 2 (400^3 fp32, R=20, 10 inner sweeps, 20 dB), seeded
synthetic data (SURVEY 8(d) generator), stopping disabled.

  python bench.py [--gpus N --steps K --warmup W --config c2 --impl ours|reference]

Prints ONE JSON line (rank 0).  ``value`` is device-timed (CUDA events on the
solver stream, max over ranks) with the tensor resident in HBM; ``e2e`` is the
same metric through the public ``fit`` API from pinned host memory with the
H2D upload and the result readback inside the timed region.  ``roofline`` is
the MTTKRP kernel's algorithmic HBM bytes / its measured launch duration.
``--impl reference`` times the reference algorithm on host cores (the CPU
oracle port in oracle/, since the reference is Python and does not travel).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--engine", default="auto", choices=["auto", "cuda_core", "tcgen05"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sharded", action="store_true",
                    help="one GPU: run the sharded engine on a one-rank NCCL group")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="diagnostic: no per-kernel events in the graph (no roofline)")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_config(w, world, engine, rho0, sharded=False):
    return {
        "workload": f"{w.name}: {w.dims[0]}x{w.dims[1]}x{w.dims[2]} {w.dtype}, R={w.rank}, "
                    f"{w.inner} inner sweeps/outer, {w.snr_db:g} dB, stopping off",
        "dims": list(w.dims), "rank": w.rank, "inner_sweeps": w.inner,
        "outer_iterations_in_config": w.outer, "rho_init": "trace((C0^T C0)*(B0^T B0))/R",
        "rho_init_value": rho0, "engine": engine,
        "parallelism": (f"slab-sharded x{world} (NCCL all-gather, graph-captured iteration)"
                        if sharded else "single-gpu"),
        "l2": "inputs larger than L2: every MTTKRP streams the whole tensor "
              f"({math.prod(w.dims) * (4 if w.dtype == 'float32' else 8) / 2**20:.0f} MiB)",
        "data": "synthetic seeded (SURVEY 8(d) generator), data seed derive_seed(0,101,0)",
    }


def cpu_oracle_rate(w, seconds: float, warm: int = 1):
    """Reference algorithm (oracle port of solver.iterate) on host cores: time
    Gauss-Seidel sweeps (3 mode updates each) for ~``seconds``; outer it/s =
    1 / (inner x sweep time).  Returns (rate, sweeps timed, unfold seconds)."""
    import numpy as np

    from oracle import ntf_oracle as O
    from paper_1409_2383_b200 import synth

    dseed, fseed = synth.seeds()
    dt = np.float32 if w.dtype == "float32" else np.float64
    x, _ = synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=dt)
    t = O.OracleTensor(x.astype(np.float64))
    del x
    t0 = time.perf_counter()
    for m in (1, 2, 3):
        t.unfolding(m)
    unfold_s = time.perf_counter() - t0
    st = O.init_state(t.dims, w.rank, O.Config(seed=fseed))
    f = list(st.factors)

    def sweep():
        for mode in (1, 2, 3):
            f[mode - 1] = O.factor_update(t, f, st.aux[mode - 1], st.duals[mode - 1],
                                          st.rho[mode - 1], mode)

    for _ in range(warm):
        sweep()
    n, t0 = 0, time.perf_counter()
    while True:
        sweep()
        n += 1
        el = time.perf_counter() - t0
        if (el >= seconds and n >= 2) or n >= 10000:
            break
    return 1.0 / (w.inner * el / n), n, unfold_s


def run_reference(args):
    """--impl reference: the reference algorithm on host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1409_2383_b200 import synth

    w = synth.CONFIGS[args.config]
    import numpy as np

    from oracle import ntf_oracle as O

    dseed, fseed = synth.seeds()
    dt = np.float32 if w.dtype == "float32" else np.float64
    x, _ = synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=dt)
    t = O.OracleTensor(x.astype(np.float64))
    del x
    for m in (1, 2, 3):
        t.unfolding(m)
    st = O.init_state(t.dims, w.rank, O.Config(seed=fseed))
    f = list(st.factors)

    def sweep():
        for mode in (1, 2, 3):
            f[mode - 1] = O.factor_update(t, f, st.aux[mode - 1], st.duals[mode - 1],
                                          st.rho[mode - 1], mode)

    for _ in range(args.warmup):
        sweep()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sweep()
    el = time.perf_counter() - t0
    rate = args.steps / (el * w.inner)
    cores = os.cpu_count()
    rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
    out = {
        "metric": "ntf_outer_iters_per_sec", "value": rate, "unit": "outer_it/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * el / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, 1, "cpu-oracle", rho0),
        "cpu_baseline": {"value": rate, "unit": "outer_it/s", "cores": cores, "kind": "port",
                         "sample": f"each step = one Gauss-Seidel sweep (3 mode updates: KR + "
                                   f"unfolding dgemm + cho_factor/cho_solve) of {w.name}; "
                                   f"outer it/s = 1/({w.inner} x sweep time); OpenBLAS threads = "
                                   f"all {cores} host cores"},
        "e2e": {"value": rate, "unit": "outer_it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1409_2383_b200 as P
    from paper_1409_2383_b200 import synth
    from paper_1409_2383_b200.engine import DeviceProblem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    elif args.sharded:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1,
                                device_id=device)
    w = synth.CONFIGS[args.config]
    engine = P.solver._engine_code(args.engine)
    dseed, fseed = synth.seeds()
    dt_np = np.float32 if w.dtype == "float32" else np.float64
    dt_t = torch.float32 if w.dtype == "float32" else torch.float64
    x_host = torch.empty(w.dims, dtype=dt_t, pin_memory=True)
    synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=dt_np, out=x_host.numpy())
    rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
    cap = args.warmup + args.steps + 1
    cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=cap, max_restarts=0,
                         inner_sweeps=w.inner, rho_init=rho0)
    if not sharded:
        x = x_host.to(device)
        prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=cap, engine=engine)
        slab_elems = [math.prod(w.dims)] * 3
        rows = list(w.dims)
    else:
        from paper_1409_2383_b200.distributed import Comm, PartitionPlan, _sharded_problem_class, make_slabs

        comm = Comm()
        plan = PartitionPlan.uniform(w.dims, world)
        slabs = make_slabs(x_host, plan, rank, device)
        prob = _sharded_problem_class()(slabs, w.dims, w.rank, cfg, cap, engine, plan, comm)
        slab_elems = [s.numel() for s in slabs]
        rows = [plan.extents[m][rank] for m in range(3)]
    st = P.init_state(w.dims, w.rank, cfg)
    prob.load_state(st.factors, st.aux, st.duals, st.rho)
    # Two captured graphs of one outer iteration: plain, and instrumented with
    # CUDA events around every MTTKRP / row update.  Warm-up captures both;
    # the timed region replays K-1 plain steps and, last, one instrumented
    # step whose per-launch times give the roofline (measured live, inside
    # the timed region, at ~no instrumentation cost to `value`).
    timed_last = not args.no_kernel_timing
    for i in range(args.warmup):
        prob.set_timing(timed_last and i == args.warmup - 1)
        prob.step()
    prob.stream.synchronize()
    if sharded:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(prob.stream)
    for i in range(args.steps):
        prob.set_timing(timed_last and i == args.steps - 1)
        prob.step()
    e1.record(prob.stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
    if sharded:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        dist.barrier()
    t_ms = float(t_ms.item())
    done, _ = prob.check_status()
    if args.no_kernel_timing:
        ktimes = np.full((w.inner * 3, 2), np.nan)
    else:
        ktimes = prob.kernel_times()  # [inner*3][2] ms, the last timed step
    # algorithmic bytes of one mode-n MTTKRP on this rank:
    # s_X * |slab| + 8 R (sum of companion extents + output rows)
    sx = 4 if w.dtype == "float32" else 8
    bytes_mode = []
    for m in range(3):
        comp = sum(w.dims[a] for a in range(3) if a != m)
        bytes_mode.append(sx * slab_elems[m] + 8 * w.rank * (comp + rows[m]))
    mt = ktimes[:, 0].reshape(w.inner, 3)
    upd = ktimes[:, 1].reshape(w.inner, 3)
    per_mode_ms = mt.mean(axis=0)
    tot_bytes = sum(bytes_mode[m] * w.inner for m in range(3))
    tot_ms = float(mt.sum())
    achieved = tot_bytes / (tot_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peak()
    step_ms = t_ms / args.steps
    value = args.steps / (t_ms * 1e-3)
    mttkrp_share = tot_ms / step_ms if step_ms > 0 else None
    prof = os.path.join(REPO, "profiles", "ncu_traffic.json")
    traffic = None
    try:
        with open(prof) as fh:
            traffic = json.load(fh).get(args.config)
    except Exception:
        traffic = None
    prob.set_timing(False)
    prob.close()  # the e2e leg below is a fresh user call: release this plan first
    del prob
    if not sharded:
        del x
    torch.cuda.synchronize()

    # ---- end to end through the public API (pinned host input) -------------
    e2e = None
    if not args.no_e2e:
        cfg_e = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer,
                               max_restarts=0, inner_sweeps=w.inner, rho_init=rho0)
        if sharded:
            def fitfn(t, r, s_, c):
                return P.distributed_fit(t, r, s_, c, sharded=True)
        else:
            fitfn = P.fit
        fitfn(P.DenseTensor(x_host), w.rank, None, cfg_e)  # warm-up
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        t0 = time.perf_counter()
        res = None
        for _ in range(args.e2e_steps):
            res = fitfn(P.DenseTensor(x_host), w.rank, None, cfg_e)
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=device)
        if sharded:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        el = float(el.item())
        h2d = x_host.numel() * x_host.element_size() + 8 * w.rank * sum(w.dims) * 3 + 24
        d2h = 8 * w.rank * sum(w.dims) * 3 + 48 * w.outer + 64
        e2e = {"value": args.e2e_steps * w.outer / el, "unit": "outer_it/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "step": (f"one fit() call of {w.outer} outer iterations from a pinned host tensor (H2D of the "
                        "tensor, block-image split, state upload, iterations, final RFE and model read-back; "
                        "back-to-back calls of one geometry reuse the plan and its graph, as the warm-up call "
                        "leaves it)"),
               "final_rfe": res.rfe}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, n, unfold_s = cpu_oracle_rate(w, args.cpu_seconds)
        cpu = {"value": rate, "unit": "outer_it/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{n} Gauss-Seidel sweeps of {w.name} (oracle port of the reference "
                         f"solver: unfolding dgemm + KR + cho_solve, OpenBLAS on all cores); "
                         f"outer it/s = 1/({w.inner} x sweep time); unfolding warm-up "
                         f"{unfold_s:.1f}s excluded"}

    if rank == 0:
        # per mode update: ridge (side stream), [W-slice], MTTKRP, row update,
        # Gram reduction (side stream); per step: 3 norm reductions + finalize
        tc = w.dtype == "float32" and w.rank <= 64 and args.engine != "cuda_core"
        launches_per_step = w.inner * 3 * (4 + (1 if tc else 0)) + 3 + 1
        if sharded:  # + Gram refresh (partial + reduce) and column maxima per mode update
            launches_per_step += w.inner * 3 * 3
        out = {
            "metric": "ntf_outer_iters_per_sec", "value": value, "unit": "outer_it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if w.dtype == "float32" else "f64", "data": "synthetic",
            "config": workload_config(w, world, args.engine, rho0, sharded),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "MTTKRP op (fp32: W-slice + tcgen05 kernels; fp64: CUDA-core kernel), all modes: "
                                   "CUDA events on the solver stream around each of the "
                                   f"{3 * w.inner} MTTKRP launches of the last timed step",
                         "per_mode_ms": [float(v) for v in per_mode_ms],
                         "per_mode_gbs": [bytes_mode[m] / (per_mode_ms[m] * 1e-3) / 1e9
                                          for m in range(3)],
                         "bytes_per_launch": bytes_mode, "mttkrp_share_of_step": mttkrp_share,
                         "row_update_ms_mean": float(upd.mean())},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches_per_step * args.steps,
            "iterations_run": done,
        }
        print(json.dumps(out), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
