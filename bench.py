#!/usr/bin/env python
"""Benchmark of the B200 RLOBPCG hot path (BASELINE.json metric, config C2).

Metric: time-to-solution (s) of rlobpcg_single on the headline configuration
(m = 1e6, n = 1e3 fp64, b = 1, d = 4n, tol 1e-12, tolerance-only stop, solver
seed 7) with A resident in HBM; one step = one complete solve (sketch, sketch
SVD, init, all LOBPCG iterations).  Also reported: the A-stream GB/s per
iteration, the roofline of the dominant kernel (the A*W pass, which in
one-pass mode also forms A^T A W) measured live with CUDA events on the
library's stream, and an end-to-end number
through the public host-buffer entry point (msvd_solve_host, pinned A copied
in every step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c5|...]
    torchrun ... bench.py --gpus N   (row-sharded over NCCL, one rank per GPU)

`--gpus N` without torchrun spawns the N ranks itself and fails if fewer than
N GPUs are visible.  Every rank generates only its own rows of A
(problems.make_problem_shard), so the global A is the same at every N.

`--impl reference` times the reference's own CPU solver (oracle/_ref, built
from the reference's sources) on the same bytes: complete solves of the FULL
configuration for C1/C2/C4 (about a minute each at C2, one thread -- the
reference has no threading), a bounded, extrapolated sample for C3/C5.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution (s) & A-stream HBM GB/s per iteration, m=1e6 n=1e3 fp64"
FALLBACK_HBM = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--m", type=int, default=0, help="override rows (debug only; invalidates the metric)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-budget", type=float, default=420.0,
                   help="--impl reference: stop timing further full solves once this many seconds are spent")
    p.add_argument("--selftest", action="store_true",
                   help="launcher/line-format check on CPU (gloo): no solve, no GPU")
    p.add_argument("--workload", default="solve", choices=["solve", "csr", "lanczos"],
                   help="solve: the BASELINE metric (default); csr / lanczos: the SURVEY 8f rows, "
                        "measured on their own lines")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append([time.perf_counter()] + parts)

    def mark(self, which):
        setattr(self, which, time.perf_counter())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        timed = [r[1:] for r in self.rows if t0 <= r[0] <= t1]
        rows = timed if len(timed) >= 3 else [r[1:] for r in self.rows]  # short window: whole run
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "samples_in_timed_region": len(timed),
                "window": "timed region" if len(timed) >= 3 else "warm-up + timed region"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_cpu():
    """CPU model and core counts of the box (the reference arm's hardware)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(), "usable_cpus": len(os.sched_getaffinity(0))}


def workload(cfg, m):
    return {"workload": f"{cfg.name}: m={m} n={cfg.n} b={cfg.b} d={cfg.d} tol={cfg.tol:g} tol-only",
            "l2": "inputs larger than L2 (A = %.1f GB)" % (8.0 * m * cfg.n / 1e9)}


# Configurations whose full-size reference solve fits a bench run (about a
# minute on one core); C3 (an SVD of 4000 x 2000, about 6 min) and
# C5 (hours, and 64 GB in host RAM) are timed on a bounded sample instead.
FULL_REFERENCE = ("c1", "c2", "c4")


def reference_solves(cfg, a_host, steps, budget_s, warmup):
    """Time the reference's own solver (oracle/_ref: minsvd compiled from its
    sources, one thread -- it has no threading) on the FULL configuration,
    A column-major in host RAM.  Each step is one complete lobpcg_solve,
    std::chrono around the call in the harness (steady_clock equivalent)
    plus the reference's own set-up time record.rows[0].wall_ms
    (solver.cpp:317-323, :382).  Steps stop early once `budget_s` is spent;
    the line reports the steps actually run."""
    from oracle import pyoracle
    from paper_2602_16797_b200 import abi, problems

    kind = "reference" if pyoracle.available("ref") else "port"
    orc = pyoracle.load("ref" if kind == "reference" else "port")
    opts = abi.default_options(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                               use_stagnation=0, record_timing=1)
    c1 = problems.CONFIGS["c1"]
    if warmup:  # page the library in: C1-size solves (0.1 s each), not the timed workload
        a1, _ = pyoracle.load("port").synth_dense(c1.spectrum(), c1.m, problems.DATA_SEED)
        for _ in range(warmup):
            orc.lobpcg_solve(a1, abi.default_options(seed=7, sketch_dim=c1.d, tol=c1.tol, use_stagnation=0))
    times, setups, r = [], [], None
    t_start = time.perf_counter()
    for k in range(steps):
        t0 = time.perf_counter()
        r = orc.lobpcg_solve(a_host, opts)
        times.append(time.perf_counter() - t0)
        setups.append(r["record"][0]["wall_ms"] / 1e3)
        if time.perf_counter() - t_start + times[-1] > budget_s:
            break
    return kind, times, setups, r


def reference_sample(cfg, steps):
    """Bounded-sample reference timing for configurations whose full CPU solve
    does not fit a bench run (C3, C5): the same recipe at m = 2e4 (full n, b,
    d), extrapolated linearly in m for the sketch and the A passes (the sketch
    SVD does not depend on m)."""
    from oracle import pyoracle
    from paper_2602_16797_b200 import abi, problems

    kind = "reference" if pyoracle.available("ref") else "port"
    orc = pyoracle.load("ref" if kind == "reference" else "port")
    m_s = 20_000
    sig = cfg.spectrum()
    a, _ = pyoracle.load("port").synth_fast(sig, m_s, problems.DATA_SEED)
    opts = abi.default_options(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                               use_stagnation=0, record_timing=1)
    vals = []
    for _ in range(max(1, min(steps, 2))):
        t0 = time.perf_counter()
        r = orc.lobpcg_solve(a, opts)
        t = time.perf_counter() - t0
        t1 = time.perf_counter()
        orc.sketch_apply(a, cfg.d, 4, problems.SOLVER_SEED)
        t_sk = time.perf_counter() - t1
        setup = r["record"][0]["wall_ms"] / 1e3
        per_pass = (t - setup) / max(1, 2 * r["iterations"])
        vals.append(t + (cfg.m / m_s - 1.0) * (t_sk + per_pass * 2 * (r["iterations"] + 1)))
    sample = (f"{kind} lobpcg_solve (one thread) on the {cfg.name} recipe at m={m_s} (full n={cfg.n}, b={cfg.b}, "
              f"d={cfg.d}), {r['iterations']} iterations, {t:.1f} s; EXTRAPOLATED to m={cfg.m} linearly in the "
              f"sketch and the A passes (the full solve does not fit a bench run)")
    return kind, vals, sample


def reference_arm(args, cfg):
    """`--impl reference`: the reference's own CPU solver on this config, on
    the box's host cores, on the same bytes our arm solves (generated on the
    device, transposed once to the reference's column-major DenseMatrix)."""
    import torch

    from paper_2602_16797_b200 import problems

    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    sig = cfg.spectrum()
    m = args.m or cfg.m
    cpu = host_cpu()
    if cfg.name in FULL_REFERENCE or args.m:
        if torch.cuda.is_available():
            a_dev, _ = problems.make_problem_shard(m, cfg.n, sig, 0, m, device="cuda:0")
            a = a_dev.t().contiguous().cpu().numpy().T  # column-major
            del a_dev
            torch.cuda.empty_cache()
        else:
            from oracle import pyoracle
            a, _ = pyoracle.load("port").synth_fast(sig, m, problems.DATA_SEED)
        kind, times, setups, r = reference_solves(cfg, a, args.steps, args.ref_budget, args.warmup)
        value = float(np.mean(times))
        iters = r["iterations"]
        per_iter = (value - float(np.mean(setups))) / max(1, iters + 1)
        a_gbs = 2 * 8.0 * m * cfg.n / per_iter / 1e9
        sample = (f"{kind} lobpcg_solve on the FULL {cfg.name} configuration (m={m}, n={cfg.n}, b={cfg.b}, "
                  f"d={cfg.d}, tol {cfg.tol:g}, tol-only), one thread (the reference has no threading), "
                  f"{len(times)} complete solve(s) of {iters} iterations; set-up (sketch + sketch SVD, "
                  f"record.rows[0].wall_ms) {np.mean(setups):.1f} s")
        steps = len(times)
        extra = {"iterations": iters, "status": r["status"], "sigma": [float(x) for x in r["sigma"]],
                 "setup_s": float(np.mean(setups)), "steps_requested": args.steps,
                 "warmup_kind": "C1-size reference solves (library page-in), untimed"}
    else:
        kind, times, sample = reference_sample(cfg, args.steps)
        value = float(np.mean(times))
        steps = len(times)
        a_gbs = None
        extra = {"steps_requested": args.steps, "extrapolated": True}
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U diag(s) V^T, generated on device)",
        "config": workload(cfg, m), "impl": "reference", "a_stream_gbs": a_gbs,
        "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": kind, "sample": sample, "host": cpu},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    line.update(extra)
    return line


def parity_vs(res, r, b, tol):
    """The north-star gates of our solve against the reference's on the same
    bytes (|dsigma| <= 1e-10 sigma_max, sin <= 1e-8 for v_min, +-1 iterations)."""
    smax = r["sigma_max_estimate"]
    ds = float(np.max(np.abs(np.asarray(res.sigma) - np.asarray(r["sigma"])))) / smax
    vr, vg = r["v"][:, 0], res.v[:, 0]
    sin = float(np.linalg.norm(vr - vg * (vg @ vr)))
    di = res.iterations() - r["iterations"]
    return {"dsigma_over_sigma_max": ds, "sin_vmin": sin, "iterations_ours": res.iterations(),
            "iterations_reference": r["iterations"], "ok": bool(ds <= 1e-10 and sin <= 1e-8 and abs(di) <= 1)}


def cpu_baseline_for(args, cfg, a, res):
    """Reported CPU baseline for our arm (rank 0, N = 1): one reference solve
    of the same bytes at the full configuration where that fits (C1, C2, C4),
    with the parity of our answer against it; a bounded sample otherwise."""
    import torch

    if cfg.name in FULL_REFERENCE or args.m:
        host = a.t().contiguous().cpu().numpy().T
        torch.cuda.empty_cache()
        kind, times, setups, r = reference_solves(cfg, host, 1, 0.0, 0)
        out = {"value": times[0], "unit": "s", "cores": 1, "kind": kind, "host": host_cpu(),
               "sample": f"one complete {kind} lobpcg_solve of the same A bytes (full {cfg.name}), one thread; "
                         f"set-up {setups[0]:.1f} s, {r['iterations']} iterations"}
        return out, parity_vs(res, r, cfg.b, cfg.tol)
    kind, vals, sample = reference_sample(cfg, 1)
    return {"value": vals[0], "unit": "s", "cores": 1, "kind": kind, "sample": sample, "host": host_cpu()}, None


def ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2602_16797_b200 import minsvd as msvd
    from paper_2602_16797_b200 import problems

    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws} (launch through torchrun, or run "
                         f"without WORLD_SIZE and bench.py spawns the ranks)")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench: rank {rank} needs GPU {local}, only {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.tensor(list(msvd.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        stream = torch.cuda.current_stream(dev)
        ctx = msvd.Context(local, comm_kind=1, nranks=ws, rank=rank, nccl_id=bytes(idt.cpu().tolist()),
                           stream=stream.cuda_stream or 1)
    else:
        stream = torch.cuda.current_stream(dev)
        ctx = msvd.Context(local, stream=stream.cuda_stream or 1)

    m = args.m or cfg.m
    sig = cfg.spectrum()
    r0, rows = msvd.shard_rows(m, ws, rank)
    # each rank generates and orthonormalises only its own rows (the R
    # factors of the generator's TSQR meet in one allreduce)
    a, vtrue = problems.make_problem_shard(m, cfg.n, sig, r0, rows,
                                           (lambda t: dist.all_reduce(t)) if ws > 1 else None, device=dev)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    op = msvd.DeviceDenseOperator(a, ctx=ctx, row0=r0, m_global=m)
    opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                              use_stagnation=False, record_timing=False)
    solve = msvd.rlobpcg_single if cfg.b == 1 else msvd.rlobpcg_block

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        res = solve(op, opts)
    barrier()
    clocks.mark("t0")
    ctx.profile(1)  # CUDA events around the A passes only: the roofline kernel, measured in the timed region
    l0 = ctx.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    iters = []
    loop_ms = []
    for _ in range(args.steps):
        res = solve(op, opts)
        iters.append(res.iterations())
        loop_ms.append(res.timings_ms["loop"])
    ev1.record(stream)
    barrier()
    clocks.mark("t1")
    launches = ctx.launch_count() - l0
    prof = ctx.profile_read()
    # per-class breakdown of every kernel (events around each launch) from
    # one more solve after the timed region
    ctx.profile(True)
    solve(op, opts)
    prof_all = ctx.profile_read()
    ctx.profile(False)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    ms_step = ms / args.steps
    it = int(np.median(iters))
    # A-stream rate of the iteration loop: passes over A actually made in the
    # loop (A*W every iteration; the Gram pass every iteration in two-pass
    # mode, at check iterations in one-pass mode) x 8 m n bytes / loop time
    per_step = (prof["apply"][1] + prof["gram"][1]) / max(1, args.steps)
    # minus the initial block's passes: A V0 and its Gram pass (two-pass mode),
    # or the one pass that forms both (one-pass mode: fewer Gram passes than
    # iterations)
    init_passes = 2 if prof["gram"][1] / max(1, args.steps) >= max(1, it) else 1
    loop_passes = per_step - init_passes
    a_gbs_iter = loop_passes * 8.0 * rows * cfg.n / (np.median(loop_ms) / 1e3) / 1e9 if it else None

    # roofline of the dominant kernel -- the A*W pass, which in one-pass mode
    # also forms A^T A W and folds the TSQR (every iteration), while the
    # stand-alone Gram pass runs only at check iterations.  Algorithmic bytes
    # per launch = 8 * m_local * n (A once; the skinny reads/writes are <0.5%).
    g_ms, g_cnt = prof["gram"]
    a_ms, a_cnt = prof["apply"]
    bytes_launch = 8.0 * rows * cfg.n
    peak, peak_kind = peaks()
    achieved_gram = bytes_launch / (g_ms / g_cnt / 1e3) / 1e9 if g_cnt else None
    achieved_apply = bytes_launch / (a_ms / a_cnt / 1e3) / 1e9 if a_cnt else None
    dominant = "apply" if a_ms >= g_ms else "gram"
    achieved = achieved_apply if dominant == "apply" else achieved_gram
    kname = ("apply kernel (K3: A W; one-pass: + A^T A W and the fused TSQR)" if dominant == "apply"
             else "gram_kernel (K2, A^T Y)")
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cfg.name, {}).get(dominant + "_kernel")
        except Exception:
            traffic = None
    smax = res.sigma_max_estimate
    truth = {"sigma_err_over_sigma_max": [float(abs(res.sigma[j] - sig[::-1][j]) / smax) for j in range(cfg.b)],
             "sin_vmin_vs_truth": float(np.linalg.norm(vtrue[:, -1] - res.v[:, 0] * (res.v[:, 0] @ vtrue[:, -1])))}

    line = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U diag(s) V^T, generated on device)",
        "config": workload(cfg, m),
        "parallelism": f"row-shard x{ws} (rows {rows} on rank 0)",
        "iterations": it, "status": res.status, "sigma": [float(x) for x in res.sigma], "vs_truth": truth,
        "a_stream_gbs_per_iter": a_gbs_iter,
        "a_passes_per_iter": loop_passes / it if it else None,
        "breakdown_ms": {k: round(v, 3) for k, v in res.timings_ms.items()},
        "kernel_ms": {k: round(v[0], 3) for k, v in prof_all.items()},
        "roofline": {"kernel": kname, "bound": "hbm", "achieved": achieved,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "frac_of_8tbs": (achieved / 8000.0) if achieved else None,
                     "bytes_per_launch": bytes_launch, "per_gpu": True,
                     "launches": a_cnt if dominant == "apply" else g_cnt,
                     "apply_kernel_achieved": achieved_apply, "gram_kernel_achieved": achieved_gram,
                     "gram_launches": g_cnt},
        "clocks": clk,
        "gpu_launches": launches,
    }
    if rank == 0 and ws == 1 and not args.no_e2e:
        line["e2e"] = e2e(msvd, ctx, a, res, opts, args, cfg, solve)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"], par = cpu_baseline_for(args, cfg, a, res)
            if par is not None:
                line["parity_vs_reference"] = par
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if ws > 1:
        dist.barrier()
    return line if rank == 0 else None


def e2e(msvd, ctx, a, res, opts, args, cfg, solve):
    """Same metric through the public host-buffer entry (msvd_solve_host):
    pinned host A copied H2D inside every step, results read back D2H."""
    import torch

    host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(a)
    hnp = host.numpy()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    msvd.solve_host(hnp, opts, ctx=ctx)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        r = msvd.solve_host(hnp, opts, ctx=ctx)
    t = (time.perf_counter() - t0) / steps
    h2d = 8 * a.shape[0] * a.shape[1]
    d2h = 8 * cfg.n * cfg.b + 64 * len(r.record.rows) + 8 * cfg.b
    del host
    return {"value": t, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "note": "wall clock around msvd_solve_host (synchronous call), pinned host A"}


def extra_workload(args, cfg):
    """Measurement lines for the SURVEY 8f rows (not the headline metric):
    csr     -- rlobpcg on a seeded sparse operator (problems.random_csr,
               m = 2e6, n = 1000, ~10 nonzeros per row, int32 indices) through
               DeviceCsrOperator; roofline of the CSR apply (SpMM) and adjoint
               (CSC gather) against their algorithmic bytes (nnz * (8 + 4) +
               8 m, + the gathered vector traffic not counted).
    lanczos -- lanczos_gk (baselines.cpp:51-166) on the C2 matrix, 200 steps
               from the randomized preconditioner's start vector (the compare
               client's run); two passes over A per step."""
    import torch

    from paper_2602_16797_b200 import minsvd as msvd
    from paper_2602_16797_b200 import problems

    dev = torch.device("cuda", 0)
    ctx = msvd.Context(0, stream=torch.cuda.current_stream(dev).cuda_stream or 1)
    peak, peak_kind = peaks()
    line = {"higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "data": "synthetic"}
    if args.workload == "csr":
        m, n, dens = args.m or 2_000_000, 1000, 0.01
        rp, ci, v = problems.random_csr(m, n, dens, 41)
        op = msvd.DeviceCsrOperator(torch.as_tensor(rp, device=dev), torch.as_tensor(ci, device=dev).to(torch.int32),
                                    torch.as_tensor(v, device=dev), n, ctx=ctx)
        opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=4 * n, tol=1e-10, use_stagnation=False,
                                  record_timing=False)
        run = lambda: msvd.rlobpcg_single(op, opts)  # noqa: E731
        nnz = int(v.size)
        work = f"csr: m={m} n={n} nnz={nnz} (density {dens:g}, int32 indices) b=1 d={4 * n} tol=1e-10 tol-only"
        bytes_pass = nnz * (8 + 4) + 8 * (m + 1)
    else:
        cfg2 = problems.CONFIGS["c2"]
        a, vmin = problems.make_problem_gpu(cfg2.m, cfg2.n, cfg2.spectrum(), device=dev)
        op = msvd.DeviceDenseOperator(a, ctx=ctx)
        opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg2.d, tol=cfg2.tol, use_stagnation=False,
                                  record_timing=False, max_iter=0)
        pre = msvd.lobpcg_solve(op, msvd.PrecondKind.randomized, opts, want_precond=True)
        v0 = msvd.sketch_and_solve_init(pre.precond, 1)[:, 0]
        iters = 200
        run = lambda: msvd.lanczos_gk(op, iters, v0, record_timing=False)  # noqa: E731
        m, n = cfg2.m, cfg2.n
        work = f"lanczos_gk: c2 matrix m={m} n={n}, {iters} steps from the rlobpcg start vector"
        bytes_pass = 8 * m * n
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    ctx.profile(1)  # events around the A passes only (the roofline kernels)
    l0 = ctx.launch_count()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = run()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / args.steps
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = (ctx.launch_count() - l0) // args.steps
    a_ms, a_cnt = prof["apply"]
    g_ms, g_cnt = prof["gram"]
    ach_a = bytes_pass / (a_ms / a_cnt / 1e3) / 1e9 if a_cnt else None
    ach_g = bytes_pass / (g_ms / g_cnt / 1e3) / 1e9 if g_cnt else None
    line.update({"metric": f"time-to-solution (s), {args.workload}", "value": t, "unit": "s",
                 "ms_per_step": t * 1e3, "config": {"workload": work},
                 "kernel_ms": {k: round(v[0] / max(1, args.steps), 3) for k, v in prof.items()},
                 "roofline": {"kernel": "apply pass (A W)" if args.workload == "lanczos" else "CSR SpMM (A W)",
                              "bound": "hbm", "achieved": ach_a, "peak": peak, "peak_kind": peak_kind,
                              "unit": "GB/s", "frac": ach_a / peak if ach_a else None,
                              "bytes_per_launch": bytes_pass, "adjoint_achieved": ach_g,
                              "adjoint_frac": ach_g / peak if ach_g else None},
                 "gpu_launches": launches})
    if args.workload == "csr":
        line["iterations"] = res.iterations()
        line["sigma_min"] = float(res.sigma[0])
    else:
        line["steps_run"] = res.steps
        line["sigma_min"] = float(res.sigma_min)
    return line


def spawn_ranks(args):
    """`--gpus N` outside a torchrun environment: launch the N ranks here
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1)
    and return their exit status.  Never downgrades to fewer ranks."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def selftest(args, cfg):
    """Launcher and line-format check without a GPU (gloo): every rank does a
    fixed CPU stand-in step; the timing is the max over ranks, as in ours()."""
    import torch
    import torch.distributed as dist

    ws, rank, _ = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if ws > 1:
        dist.init_process_group("gloo")
    x = torch.ones(128, 128, dtype=torch.float64)
    for _ in range(args.warmup):
        x @ x
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x @ x
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item() * 1e3 / args.steps
    line = {"metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "selftest (no solve)", "config": workload(cfg, cfg.m),
            "parallelism": f"row-shard x{ws}", "selftest": True, "ranks_reported": ws}
    if ws > 1:
        dist.destroy_process_group()
    return line if rank == 0 else None


def main():
    args = parse()
    from paper_2602_16797_b200 import problems

    cfg = problems.CONFIGS[args.config]
    if args.workload != "solve":
        print(json.dumps(extra_workload(args, cfg)), flush=True)
        return
    if args.impl == "reference":
        line = reference_arm(args, cfg)  # rank 0 only; the others exit without work
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if not args.selftest:
            import torch

            have = torch.cuda.device_count()
            if have < args.gpus:
                raise SystemExit(f"bench: --gpus {args.gpus} needs {args.gpus} GPUs, {have} visible")
        sys.exit(spawn_ranks(args))
    line = selftest(args, cfg) if args.selftest else ours(args, cfg)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
