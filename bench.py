#!/usr/bin/env python
"""Benchmark: NTF outer iterations/sec on B200 (BASELINE.json metric).

One *step* is one ADMoM outer iteration of the reference algorithm
(solver.iterate, reference solver.py:295-327): ``inner`` Gauss-Seidel sweeps
x 3 modes of (dense MTTKRP -> ridge Cholesky -> row solve), with the
projection / dual step / residuals / adaptation fused in.  Default workload:
BASELINE config 5 (2000^3 fp32 = 32 GB, R=100, 5 inner sweeps, 20 dB), the
largest configuration that fits one GPU, with seeded synthetic data generated
in HBM by the counter-based generator (synth.py; the bytes the oracle
restates), stopping disabled.  ``--config c1..c4`` selects the others.

  python bench.py [--gpus N --steps K --warmup W --config c5 --impl ours|reference]

Prints ONE JSON line (rank 0).  ``value`` is device-timed (CUDA events on the
solver stream, max over ranks) with the tensor resident in HBM; ``e2e`` is the
same metric through the public ``fit`` / ``distributed_fit`` API from pinned
host memory with the H2D upload and the result readback inside the timed
region.  ``roofline`` is the MTTKRP's algorithmic HBM bytes over its launch
durations, from the last timed step, which is launched without programmatic
dependent launch (serialised kernels) so the per-kernel CUDA events cannot
overlap.  ``--impl reference`` times the reference algorithm on host cores
(the CPU oracle port in oracle/, since the reference is Python and does not
travel) on a bounded sample of the same workload.
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
# Environment variables that select diagnostic code or another library: a
# timed run refuses them (release libraries ignore the diagnostic ones anyway).
FORBIDDEN_ENV_PREFIXES = ("NTF_TC_", "NTF_UPD_", "NTF_VARIANT_LIB", "NTF_B200_LIB", "NTF_B200_FUSED_RIDGE",
                          "NTF_B200_PLAN_TIMING", "NTF_DIAG")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--engine", default="auto", choices=["auto", "cuda_core", "tcgen05"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--sharded", action="store_true",
                    help="one GPU: run the sharded engine on a one-rank NCCL group")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="diagnostic: no per-kernel events in the graph (no roofline)")
    return ap.parse_args()


def check_env():
    bad = sorted(k for k in os.environ if k.startswith(FORBIDDEN_ENV_PREFIXES))
    if bad:
        sys.exit(f"bench.py: refusing to run with diagnostic/library overrides set: {bad}")
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("NTF_")}


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
                    f"{w.inner} inner sweeps/outer, {w.snr_db:g} dB"
                    f"{', 20% zeroed factor entries' if w.zero_frac else ''}, stopping off",
        "dims": list(w.dims), "rank": w.rank, "inner_sweeps": w.inner,
        "outer_iterations_in_config": w.outer, "rho_init": "trace((C0^T C0)*(B0^T B0))/R",
        "rho_init_value": rho0, "engine": engine,
        "parallelism": (f"slab-sharded x{world} (row all-gather per mode update, graph-captured iteration)"
                        if sharded else "single-gpu"),
        "l2": "inputs larger than L2: every MTTKRP streams the whole tensor "
              f"({math.prod(w.dims) * (4 if w.dtype == 'float32' else 8) / 2**20:.0f} MiB)",
        "data": "synthetic seeded counter-based generator (synth.py / csrc/synth.cu, restated in "
                "oracle/synth_oracle.c), data seed derive_seed(0,101,0)",
    }


# ---------------------------------------------------------------------------
# CPU reference algorithm on a bounded sample of the workload
# ---------------------------------------------------------------------------


class CpuSample:
    """The oracle port of the reference solver (unfolding dgemm + materialised
    Khatri-Rao + cho_solve, OpenBLAS on every host core) on the first ``I_s``
    mode-1 rows of the workload's tensor (byte-identical to those rows of the
    GPU's tensor), sized so X and its three cached unfoldings stay under
    ~8 GB.  Per-sweep cost is extrapolated to the full tensor term by term:
    the mode-1 Khatri-Rao product (C o B: J K rows) does not depend on I and
    is counted once; everything else (mode-1 GEMM and row solve, modes 2 and
    3 whose Khatri-Rao rows and GEMMs have I_s rows) scales with I / I_s."""

    def __init__(self, w, max_elems: float = 2.5e8):
        import numpy as np

        from oracle import ntf_oracle as O

        self.O = O
        self.w = w
        I, J, K = w.dims
        self.I_s = int(min(I, max(1, max_elems // (J * K))))
        self.scale = I / self.I_s
        dseed, fseed = O.derive_seed(0, O.DATA_SALT, 0), O.derive_seed(0, O.FIT_SALT, 0)
        truth = O.true_factors(w.dims, w.rank, dseed, w.zero_frac)
        sigma, key = O.noise_sigma(truth, w.snr_db), O.synth_key(dseed)
        dt = np.float32 if w.dtype == "float32" else np.float64
        t0 = time.perf_counter()
        xs = O.synth_box_c(truth, w.dims, (0, 0, 0), (self.I_s, J, K), sigma, key, dt)
        self.t = O.OracleTensor(xs.astype(np.float64))
        del xs
        for m in (1, 2, 3):
            self.t.unfolding(m)
        self.setup_s = time.perf_counter() - t0
        st = O.init_state(self.t.dims, w.rank, O.Config(seed=fseed))
        self.st = st
        self.f = list(st.factors)

    def sweep(self):
        """One Gauss-Seidel sweep; returns (seconds per mode update, KR1 seconds)."""
        O, st, f = self.O, self.st, self.f
        tm = []
        for mode in (1, 2, 3):
            t0 = time.perf_counter()
            f[mode - 1] = O.factor_update(self.t, f, st.aux[mode - 1], st.duals[mode - 1],
                                          st.rho[mode - 1], mode)
            tm.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        O.khatri_rao([f[2], f[1]])  # the mode-1 Khatri-Rao product alone
        kr1 = time.perf_counter() - t0
        return tm, kr1

    def full_sweep_seconds(self, tm, kr1) -> float:
        if self.I_s == self.w.dims[0]:
            return sum(tm)
        kr1 = min(kr1, tm[0])
        return kr1 + (tm[0] - kr1) * self.scale + (tm[1] + tm[2]) * self.scale

    def describe(self) -> str:
        I, J, K = self.w.dims
        if self.I_s == I:
            return f"the whole {self.w.name} tensor"
        return (f"the first {self.I_s} of {I} mode-1 rows of {self.w.name} ({self.I_s}x{J}x{K}, the "
                f"same bytes as the GPU tensor's rows); per-sweep time extrapolated term by term: mode-1 "
                f"Khatri-Rao (JK x R, independent of I) once, the rest x{self.scale:.2f}")


def cpu_oracle_rate(w, seconds: float):
    s = CpuSample(w)
    s.sweep()  # warm
    fulls, n, t0 = [], 0, time.perf_counter()
    while True:
        tm, kr1 = s.sweep()
        fulls.append(s.full_sweep_seconds(tm, kr1))
        n += 1
        if (time.perf_counter() - t0 >= seconds and n >= 2) or n >= 10000:
            break
    sweep = statistics.median(fulls)
    return 1.0 / (w.inner * sweep), n, s


def run_reference(args):
    """--impl reference: the reference algorithm on host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1409_2383_b200 import synth

    w = synth.CONFIGS[args.config]
    s = CpuSample(w)
    for _ in range(args.warmup):
        s.sweep()
    fulls, t0 = [], time.perf_counter()
    for _ in range(args.steps):
        tm, kr1 = s.sweep()
        fulls.append(s.full_sweep_seconds(tm, kr1))
    el = time.perf_counter() - t0
    rate = 1.0 / (w.inner * statistics.median(fulls))
    cores = os.cpu_count()
    rho0 = synth.initial_rho_trace(w.dims, w.rank, synth.seeds()[1])
    sample = (f"each step = one Gauss-Seidel sweep (3 mode updates: KR + unfolding dgemm + "
              f"cho_factor/cho_solve) of {s.describe()}; outer it/s = 1/({w.inner} x median full "
              f"sweep time); OpenBLAS threads = all {cores} host cores; sample setup "
              f"{s.setup_s:.1f}s excluded")
    out = {
        "metric": "ntf_outer_iters_per_sec", "value": rate, "unit": "outer_it/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * el / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, 1, "cpu-oracle", rho0),
        "cpu_baseline": {"value": rate, "unit": "outer_it/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "outer_it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def main():
    args = parse_args()
    env = check_env()
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
    dt = "float32" if w.dtype == "float32" else "float64"
    spec = synth.SynthSpec.of(w, dseed)
    rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
    cap = args.warmup + args.steps + 1
    cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=cap, max_restarts=0,
                         inner_sweeps=w.inner, rho_init=rho0)
    # every rank generates only its own slabs, straight into HBM
    if not sharded:
        x = synth.generate_box(spec, dtype=dt, device=device)
        prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=cap, engine=engine)
        slabs = [x]
        slab_elems = [math.prod(w.dims)] * 3
        rows = list(w.dims)
    else:
        from paper_1409_2383_b200.distributed import Comm, PartitionPlan, ShardedTensor, _sharded_problem_class

        comm = Comm()
        plan = PartitionPlan.uniform(w.dims, world)
        slabs = [synth.generate_box(spec, lo, hi, dt, device=device)
                 for lo, hi in ShardedTensor.slab_boxes(w.dims, plan, rank)]
        prob = _sharded_problem_class()(slabs, w.dims, w.rank, cfg, cap, engine, plan, comm)
        slab_elems = [s.numel() for s in slabs]
        rows = [plan.extents[m][rank] for m in range(3)]
    st = P.init_state(w.dims, w.rank, cfg)
    prob.load_state(st.factors, st.aux, st.duals, st.rho)
    # Two captured graphs of one outer iteration: plain (PDL chain), and
    # instrumented: CUDA events around every MTTKRP / row update, kernels
    # launched without PDL so each event pair brackets exactly its kernels.
    # Warm-up captures both; the timed region replays K-1 plain steps and,
    # last, one instrumented step whose per-launch times give the roofline.
    timed_last = not args.no_kernel_timing
    for i in range(args.warmup):
        prob.set_timing(timed_last and i == args.warmup - 1)
        prob.step()
    if sharded:
        prob.precapture()  # the plain graph too (captured lazily otherwise: inside the timed region)
    prob.stream.synchronize()
    if sharded:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e_last = torch.cuda.Event(enable_timing=True)  # start of the instrumented (last) step
    torch.cuda.synchronize()
    e0.record(prob.stream)
    for i in range(args.steps):
        prob.set_timing(timed_last and i == args.steps - 1)
        if i == args.steps - 1:
            e_last.record(prob.stream)
        prob.step()
    e1.record(prob.stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
    if sharded:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        dist.barrier()
    t_ms = float(t_ms.item())
    last_ms = e_last.elapsed_time(e1)  # the instrumented step alone (no PDL overlap)
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
    value = args.steps / (t_ms * 1e-3)  # outer iterations of the whole (sharded) job per second
    # share of the instrumented step itself (its kernels serialised): <= 1
    mttkrp_share = tot_ms / last_ms if last_ms > 0 else None
    traffic = None
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(args.config)
        if tr is not None and not sharded:
            traffic = tr["bytes_per_launch"]
    except Exception:
        traffic = None
    prob.set_timing(False)
    prob.close()  # the e2e leg below is a fresh user call: release this plan first
    del prob

    # ---- end to end through the public API (pinned host input) -------------
    e2e = None
    if not args.no_e2e:
        host = [torch.empty(sl.shape, dtype=sl.dtype, pin_memory=True) for sl in slabs]
        for h, sl in zip(host, slabs):
            h.copy_(sl)
        del slabs, sl
        if not sharded:
            del x
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        cfg_e = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer,
                               max_restarts=0, inner_sweeps=w.inner, rho_init=rho0)
        if sharded:
            from paper_1409_2383_b200.distributed import ShardedTensor

            def call():
                return P.distributed_fit(ShardedTensor(w.dims, plan, rank, host), w.rank, None, cfg_e,
                                         sharded=True, engine=engine)
        else:
            def call():
                return P.fit(P.DenseTensor(host[0]), w.rank, None, cfg_e, engine=engine)
        n_e2e = args.e2e_steps or (2 if math.prod(w.dims) > 2e9 else 3)
        # fit() picking another engine than the one `value` was measured on (its
        # block images not fitting the free HBM) would make e2e a different metric
        import warnings
        warnings.filterwarnings("error", message=".*block images need.*", category=RuntimeWarning)
        call()  # warm-up
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        t0 = time.perf_counter()
        res = None
        for _ in range(n_e2e):
            res = call()
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=device)
        if sharded:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        el = float(el.item())
        h2d = sum(h.numel() * h.element_size() for h in host) + 8 * w.rank * sum(w.dims) * 3 + 24
        d2h = 8 * w.rank * sum(w.dims) * 3 + 48 * w.outer + 64
        e2e = {"value": n_e2e * w.outer / el, "unit": "outer_it/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "step": (f"one {'distributed_fit' if sharded else 'fit'}() call of {w.outer} outer "
                        "iterations from pinned host memory (H2D of the tensor"
                        f"{' slabs' if sharded else ''}, block-image split, state upload, iterations, "
                        "final RFE and model read-back)"),
               "calls": n_e2e, "final_rfe": res.rfe}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, n, s = cpu_oracle_rate(w, args.cpu_seconds)
        cpu = {"value": rate, "unit": "outer_it/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{n} Gauss-Seidel sweeps of {s.describe()} (oracle port of the reference "
                         f"solver: unfolding dgemm + KR + cho_solve, OpenBLAS on all cores); "
                         f"outer it/s = 1/({w.inner} x median full-sweep time); sample setup "
                         f"{s.setup_s:.1f}s excluded"}

    if rank == 0:
        # per mode update: ridge (side stream), [W-slice], MTTKRP, row update,
        # Gram reduction (side stream); per step: 3 norm reductions + finalize
        tc = w.dtype == "float32" and args.engine != "cuda_core"
        launches_per_step = w.inner * 3 * (4 + (1 if tc else 0)) + 3 + 1
        if sharded and world > 1 and os.environ.get("NTF_B200_P2P", "0") in ("1", "force"):
            launches_per_step += w.inner * 3  # + the peer row-gather kernel per mode update
        out = {
            "metric": "ntf_outer_iters_per_sec", "value": value, "unit": "outer_it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if w.dtype == "float32" else "f64", "data": "synthetic",
            "config": workload_config(w, world, args.engine, rho0, sharded),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "MTTKRP op (fp32: W-slice + tcgen05 kernels; fp64 / engine cuda_core: the fp64-arithmetic DMMA kernel), all modes: "
                                   "CUDA events on the solver stream around each of the "
                                   f"{3 * w.inner} MTTKRP launches of the last timed step (kernels "
                                   "serialised, no PDL overlap)",
                         "per_mode_ms": [float(v) for v in per_mode_ms],
                         "per_mode_gbs": [bytes_mode[m] / (per_mode_ms[m] * 1e-3) / 1e9
                                          for m in range(3)],
                         "bytes_per_launch": bytes_mode, "mttkrp_share_of_step": mttkrp_share,
                         "instrumented_step_ms": last_ms,
                         "row_update_ms_mean": float(upd.mean())},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches_per_step * args.steps,
            "iterations_run": done, "env": env,
        }
        if cpu is None and world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = {"value": None, "note": "not run"}
        print(json.dumps(out), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
