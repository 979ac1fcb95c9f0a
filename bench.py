#!/usr/bin/env python
"""Benchmark: ASADMM iterations/s on the BASELINE config-2 workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--no-cpu-baseline] [--ttt]

A step is one ASADMM iteration of the whole problem: staged screening
(+ compaction and factor downdate when pixels freeze), the Q sensor local
updates (forward matvec, capacitance-inverse apply, adjoint matvec fused with
the x-update), the exchange (N > 1) and the fusion / stopping rule.

Workload (BASELINE.json configs[1]): Q=8 sensors, M=8, K=256 (KM=2048),
128x128 grid (N=16384), dechirped-LFM complex64 operators generated on the
GPU from seeded geometry/phases (268 MB per sensor, 2.15 GB total -- inputs
far larger than the 126 MB L2, so no L2 flush is needed between steps),
60 seeded targets, 20 dB AWGN (bit-exact reference noise stream),
mu=1, beta=rho=1, lambda = 0.05 max|A^H y|, eps_rel=1e-5, eps_abs=1e-12.

One JSON line (rank 0): value = whole-job iterations/s over K timed
iterations after W warm-up iterations, device-timed with CUDA events on the
library stream (max over ranks); e2e = the same metric through the public
API with host (pinned) buffers, H2D of the operators + setup + the solve +
D2H of the results inside the timed region; roofline = the dominant kernel's
algorithmic bytes / its average device time vs the measured HBM peak;
cpu_baseline = the fp64 CPU oracle on a bounded sample of the same workload.
--impl reference times the CPU reference path (the oracle restatement;
the reference itself cannot be built here).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance run")
    p.add_argument("--ttt-max-iter", type=int, default=3000)
    p.add_argument("--stress", action="store_true", help="BASELINE config 4 elimination-stress report")
    p.add_argument("--stress-iters", type=int, default=400)
    p.add_argument("--frames", type=int, default=0, help="BASELINE config 5: F frames sharing the operators")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=5)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(phase: str, config: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    entry = d.get(config, {}).get(phase)
    return None if entry is None else entry.get("dram_bytes_per_launch")


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def build_workload(cfg, solver, q_begin: int, q_end: int, dist=None):
    """Operators on the device; scene + bit-exact noise on the host; y = A x + w
    via the device forward operator; lambda = frac * max |A^H y| (all ranks)."""
    from paper_2307_08606_b200 import scenario
    from paper_2307_08606_b200.rng import ComplexGaussian, mix_seed
    pix, tx, rx = scenario.baseline_geometry(cfg)
    per_sensor = scenario.baseline_scene(cfg)
    ys = []
    lam_local = 0.0
    for q in range(q_begin, q_end):
        solver.generate_dechirp_operator(q - q_begin, cfg.M, cfg.K, pix, tx[q], rx[q],
                                         scenario.baseline_phases(cfg, q), cfg.fc, cfg.bw, cfg.pulse)
        y = solver.apply(q - q_begin, per_sensor[q].astype(np.complex128))
        power = float(np.vdot(y, y).real)
        sigma = math.sqrt(power / (cfg.KM * 10.0 ** (cfg.snr_db / 10.0)))
        y = y + sigma * ComplexGaussian(mix_seed(cfg.seed, q + 1)).draw(cfg.KM)
        solver.set_measurement(q - q_begin, y)
        ys.append(y)
        lam_local = max(lam_local, float(np.abs(solver.apply_adjoint(q - q_begin, y)).max()))
    if dist is not None:
        import torch
        t = torch.tensor([lam_local], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        lam_local = float(t.item())
    return ys, cfg.lambda_frac * lam_local


def algorithmic_bytes_per_iteration(cfg, sizes):
    """Dual form: 2 passes over the active columns + the Hermitian triangle of
    the KM x KM capacitance inverse (c128, KM(KM+1)/2 entries) + O(N) vectors
    (SURVEY 8d)."""
    km = cfg.KM
    return sum(2.0 * km * n * 8 + km * (km + 1) * 8 for n in sizes) + 12.0 * cfg.N * 16


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle; bounded sample)
# ---------------------------------------------------------------------------
def cpu_sample(cfg, iters: int, sample_sensors: int = 2, budget_s: float = 20.0):
    """fp64 oracle (NumPy/SciPy, all BLAS threads) on `sample_sensors` of the Q
    sensors: time `iters` local updates + the fusion round; extrapolate the
    per-sensor cost x Q (the Jacobi sweep is a sum of independent per-sensor
    solves, admm.hpp:389-390).  Setup (Woodbury factor) is excluded."""
    from oracle import admm_ref
    from paper_2307_08606_b200 import scenario
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1])
    except Exception:
        cores = os.cpu_count() or 1
    per_sensor = scenario.baseline_scene(cfg)
    h = admm_ref.Hyper(mu=cfg.mu, lambda_=1.0, beta=cfg.beta, eps_abs=cfg.eps_abs, eps_rel=cfg.eps_rel,
                       max_iter=iters)
    sensors = []
    for q in range(sample_sensors):
        a = scenario.baseline_operator(cfg, q).astype(np.complex128)
        y = scenario.simulate_measurement(a, per_sensor[q], cfg.snr_db,
                                          scenario.mix_seed(cfg.seed, q + 1))[0]
        sensors.append(admm_ref.SensorRef(a, y, h))
    fusion = admm_ref.FusionRef(cfg.N, cfg.Q, h)
    t_local = 0.0
    t_fusion = 0.0
    done = 0
    for _ in range(iters):  # bounded: stops once ~budget_s of CPU work is timed
        if done and t_local + t_fusion > budget_s:
            break
        done += 1
        t0 = time.perf_counter()
        for s in sensors:
            s.local_update(fusion.gap, fusion.sigma)
        t1 = time.perf_counter()
        for q, s in enumerate(sensors):
            fusion.set_contribution(q + 1, s.active, s.x_hat)
        fusion.round()
        t2 = time.perf_counter()
        t_local += t1 - t0
        t_fusion += t2 - t1
    iters = done
    per_iter = (t_local / sample_sensors) * cfg.Q / iters + t_fusion / iters
    # one more iteration of one sensor on a single BLAS thread (SURVEY 8d asks
    # for the 1-thread figure next to the all-core one)
    one = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            sensors[0].local_update(fusion.gap, fusion.sigma)
            t1 = time.perf_counter()
            fusion.round()
            t2 = time.perf_counter()
        one = 1.0 / ((t1 - t0) * cfg.Q + (t2 - t1))
    except Exception:
        pass
    # the headline CPU number is the faster of the two (at small shapes BLAS
    # threading overhead makes one thread faster)
    best_one = one is not None and one > 1.0 / per_iter
    return {"value": one if best_one else 1.0 / per_iter, "unit": "iterations/s",
            "cores": 1 if best_one else int(cores), "kind": "port",
            "value_all_threads": 1.0 / per_iter, "threads_all": int(cores), "value_1thread": one,
            "sample": (f"fp64 NumPy/SciPy oracle (Woodbury form), {sample_sensors} of {cfg.Q} sensors x {iters} "
                       f"iterations timed, per-sensor local-update time x{cfg.Q} + fusion; "
                       f"setup excluded; {cfg.name} shapes")}


def workload_config(cfg, world, lam, parallelism=None):
    """The config object both arms print (same workload, same keys)."""
    return {"workload": f"BASELINE {cfg.name}: Q={cfg.Q} M={cfg.M} K={cfg.K} KM={cfg.KM} "
                        f"N={cfg.N} ({cfg.nside}x{cfg.nside}), {cfg.n_targets} targets, {cfg.snr_db} dB",
            "global_batch": cfg.Q, "parallelism": parallelism or f"sensor-sharded x{world}",
            "l2": f"operators {cfg.Q * cfg.KM * cfg.N * 8 / 1e9:.2f} GB >> 126 MB L2 "
                  "(streamed every iteration; no flush needed)",
            "hyper": {"mu": cfg.mu, "beta": cfg.beta, "lambda": lam if lam is not None else "0.05 max|A^H y|",
                      "eps_rel": cfg.eps_rel, "eps_abs": cfg.eps_abs, "W": 5, "tol": 1e-5}}


def reference_arm(args, cfg):
    from paper_2307_08606_b200.distributed import env_rank_world
    rank, world, _ = env_rank_world()
    if world > 1 and rank != 0:
        return
    base = cpu_sample(cfg, max(1, args.steps))
    v = base["value"]
    out = {"metric": "ASADMM iterations/s", "value": v, "unit": "iterations/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "dtype_note": "complex128 arithmetic (fp64 NumPy/SciPy oracle)",
           "data": "synthetic (seeded BASELINE dechirp operators, host generator)",
           "impl": "reference",
           "config": workload_config(cfg, 1, lam=None, parallelism=f"host BLAS threads ({base['cores']})"),
           "cpu_baseline": {"kind": base["kind"], "cores": base["cores"], "sample": base["sample"], "value": v,
                            "unit": "iterations/s"},
           "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def ours(args, cfg):
    import torch
    from paper_2307_08606_b200 import api, distributed as D
    import __graft_entry__
    __graft_entry__.build()
    rank, world, local = D.env_rank_world()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("gloo")
        dist = tdist
    torch.cuda.set_device(local)
    uid = D.broadcast_unique_id(rank, world)
    q0, q1 = D.shard_range(cfg.Q, rank, world)
    solver = D.sharded_solver(cfg.N, cfg.Q, rank, world, local, uid) if world > 1 else api.Solver(cfg.N, cfg.Q, local)
    ys, lam = build_workload(cfg, solver, q0, q1, dist)
    W, K = args.warmup, args.steps
    hyper = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=cfg.eps_abs, eps_rel=cfg.eps_rel,
                            screening_window=5, screening_tol=1e-5, max_iter=W + K)

    # ---- timed run: W warm-up + K timed iterations, device-timed ----------
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    res = solver.run(hyper, api.Mode.ASADMM, fixed_iterations=True, fetch=False)
    clk = clocks.stop()
    torch.cuda.synchronize()
    it_ms, it_launch = solver.iteration_stats(res.iterations)
    timed_ms = float(np.sum(it_ms[W:W + K]))
    launches = int(np.sum(it_launch[W:W + K]))
    if dist is not None:
        t = torch.tensor([timed_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        timed_ms = float(t.item())
    value = K / (timed_ms / 1000.0)

    # ---- profiling pass: per-phase device time + algorithmic bytes ----------
    solver.set_profiling(True)
    solver.run(hyper, api.Mode.ASADMM, fixed_iterations=True, fetch=False)
    phases = solver.phase_stats()
    solver.set_profiling(False)
    peak, peak_kind = measured_peaks()
    kern = max(("forward", "adjoint", "gapply", "primal", "sweep"), key=lambda p: phases[p]["ms"])
    ph = phases[kern]
    per_launch_ms = ph["ms"] / max(1, ph["calls"])
    per_launch_bytes = ph["bytes"] / max(1, ph["calls"])
    achieved = per_launch_bytes / (per_launch_ms / 1000.0) / 1e9
    roofline = {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_kind,
                "traffic": ncu_traffic(kern, cfg.name),
                "algorithmic_bytes_per_launch": per_launch_bytes, "avg_launch_ms": per_launch_ms,
                "phases": {k: {"ms_per_call": v["ms"] / max(1, v["calls"]),
                               "GBps": (v["bytes"] / (v["ms"] / 1000.0) / 1e9) if v["ms"] > 0 else None,
                               "share": v["ms"] / max(1e-9, sum(p["ms"] for p in phases.values()))}
                           for k, v in phases.items() if v["calls"]}}

    # ---- time to tolerance ------------------------------------------------
    ttt, ttt_hyper = None, None
    if not args.no_ttt:
        clocks_ttt = ClockSampler(local)
        clocks_ttt.start()
        ttt, ttt_hyper = time_to_tolerance(solver, hyper, args.ttt_max_iter)
        ttt["clocks"] = clocks_ttt.stop()
    solver.close()

    # ---- e2e through the public API with pinned host buffers ---------------
    # One step = one api.run() solve to tolerance (the call a user makes):
    # H2D of the operators + setup + every iteration + D2H of every result.
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(cfg, ttt_hyper or hyper, ys, to_tolerance=ttt_hyper is not None, q0=q0, q1=q1, dist=dist)

    # ---- CPU baseline ------------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(cfg, 12, budget_s=12.0)  # about 10-15 s of CPU work
        if ttt is not None:
            ttt["cpu_oracle_time_to_tolerance_s_est"] = ttt["iterations"] / cpu["value"]

    bytes_iter = algorithmic_bytes_per_iteration(cfg, [cfg.N] * cfg.Q)
    if rank == 0:
        out = {"metric": "ASADMM iterations/s", "value": value, "unit": "iterations/s", "n_gpus": world,
               "steps": K, "warmup": W, "ms_per_step": timed_ms / K, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64", "dtype_note": "complex64 operator storage, complex128 (fp64) arithmetic; Gram from exact int8 slices",
               "data": "synthetic (seeded BASELINE dechirp operators generated on device)",
               "config": workload_config(cfg, world, lam),
               "gpu_launches": launches, "clocks": clk, "roofline": roofline,
               "iteration_GBps_algorithmic": bytes_iter * value / 1e9,
               "cpu_baseline": cpu, "e2e": e2e, "time_to_tolerance": ttt,
               "refinement": {"km_space_refinement": True, "sensors_unrefined": res.refine_skipped},
               "active_sizes_end": None}
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def time_to_tolerance(solver, hyper, max_iter):
    """Time-to-tolerance for "ASADMM to rel. residual 1e-5" (BASELINE config 2).

    With the literal mapping (eps_rel = 1e-5, eps_abs = 1e-12) the degenerate
    BASELINE problem (x_G = 0) never meets the stopping
    rule, so the residual is read as relative to the first iteration's:
    eps_abs is set so that sqrt(N) eps_abs = 1e-5 * pri_res(1), i.e. the run
    stops once the primal residual has dropped 1e5-fold (the reference's own
    stopping rule, admm.hpp:248-255, then applies unchanged)."""
    from paper_2307_08606_b200 import api
    first = solver.run(api.Hyperparams(**{**hyper.__dict__, "max_iter": 1}), api.Mode.ASADMM, fetch=True)
    pri1 = first.report.iterations[0].pri_res
    eps_abs = 1e-5 * pri1 / math.sqrt(solver.N)
    h2 = api.Hyperparams(**{**hyper.__dict__, "max_iter": max_iter, "eps_abs": eps_abs})
    r2 = solver.run(h2, api.Mode.ASADMM, fetch=True)
    ms2, _ = solver.iteration_stats(r2.iterations)
    last = r2.report.iterations[-1]
    return ({"converged": r2.converged, "iterations": r2.iterations, "solve_s_device": float(np.sum(ms2)) / 1e3,
             "setup_s": r2.setup_ms / 1e3, "time_to_tolerance_s": float(np.sum(ms2)) / 1e3 + r2.setup_ms / 1e3,
             "rule": "pri_res <= 1e-5 * pri_res(1) (eps_abs = %.3e, eps_rel = %g)" % (eps_abs, hyper.eps_rel),
             "final_pri_res": last.pri_res, "max_iter": max_iter,
             "active_sizes_end": last.active_sizes}, h2)


def e2e_run(cfg, hyper, ys, to_tolerance=True, q0=0, q1=None, dist=None, reps=3):
    """The public call a user makes, with the operators in pinned host memory:
    api.run(problem, hyper, ASADMM) on one GPU, run_distributed (every rank
    passes the Problem and uploads its own sensors, runtime.hpp:768-775)
    under torchrun.  H2D of A + y, initial factorization, the iterations (to
    tolerance) and D2H of every RunResult field are inside the timed region
    (CUDA events; max over ranks; bytes summed over ranks)."""
    import torch
    from paper_2307_08606_b200 import api, scenario, distributed as D
    q1 = cfg.Q if q1 is None else q1
    nloc = q1 - q0
    world = dist.get_world_size() if dist is not None else 1
    pinned = torch.empty((nloc, cfg.N, cfg.KM), dtype=torch.complex64, pin_memory=True)
    gen = api.Solver(cfg.N, nloc, torch.cuda.current_device())
    pix, tx, rx = scenario.baseline_geometry(cfg)
    for q in range(q0, q1):
        gen.generate_dechirp_operator(q - q0, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                      cfg.fc, cfg.bw, cfg.pulse)
        pinned[q - q0].numpy()[:] = gen.get_operator(q - q0).T
    gen.close()
    # sensors owned by other ranks: shape-only placeholders (never uploaded here)
    hole = np.broadcast_to(np.zeros((1, 1), dtype=np.complex64), (cfg.KM, cfg.N))
    ops = [api.ForwardOperator.from_matrix(pinned[q - q0].numpy().T if q0 <= q < q1 else hole)
           for q in range(cfg.Q)]  # F-contiguous views of the pinned buffers
    ys_all = [ys[q - q0] if q0 <= q < q1 else np.zeros(cfg.KM, dtype=np.complex128) for q in range(cfg.Q)]
    prob = api.Problem(ops, ys_all)
    runs = [_e2e_once(api, D, torch, prob, hyper, ys, ops, to_tolerance, q0, q1, dist, world) for _ in range(reps)]
    runs.sort(key=lambda r: r["ms"])
    med = dict(runs[len(runs) // 2])
    med["repeats"] = {"n": reps, "statistic": "median of independent api.run calls (each a fresh context)",
                      "values": sorted(r["value"] for r in runs)}
    return med


def _e2e_once(api, D, torch, prob, hyper, ys, ops, to_tolerance, q0, q1, dist, world):
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    if world == 1:  # api.run(prob, hyper, ASADMM), spelled out so each stage can be timed
        prob.validate()
        hyper.validate()
        solver = api.Solver.from_problem(prob)
        t1 = time.perf_counter()
        try:
            r = solver.run(hyper, api.Mode.ASADMM, fixed_iterations=not to_tolerance)
            t2 = time.perf_counter()
        finally:
            solver.close()
    else:
        t1 = t0
        r = D.run_distributed(prob, hyper, api.Mode.ASADMM, fixed_iterations=not to_tolerance)
        t2 = time.perf_counter()
    t3 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    h2d = sum(ops[q].matrix().nbytes for q in range(q0, q1)) + sum(np.asarray(y).nbytes for y in ys)
    d2h = (r.image.nbytes + 4 * r.x_global.nbytes + sum(x.nbytes for x in r.sensor_images)
           + sum(a.nbytes for a in r.active_sets))
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        b = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64)
        dist.all_reduce(b, op=dist.ReduceOp.SUM)
        h2d, d2h = int(b[0].item()), int(b[1].item())
    return {"value": r.iterations / (ms / 1000.0), "unit": "iterations/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "step": f"one {'api.run' if world == 1 else 'run_distributed'} call "
                    f"({'to tolerance' if to_tolerance else 'fixed'}; {r.iterations} iterations, "
                    f"converged={r.converged})",
            "ms": ms, "setup_ms": r.setup_ms, "solve_ms": r.solve_ms,
            "stages_ms": {"context_and_upload": 1e3 * (t1 - t0), "run_and_fetch": 1e3 * (t2 - t1),
                          "close": 1e3 * (t3 - t2)}}


def stress(args):
    """BASELINE config 4 (elimination stress): config-2 geometry at 0.1% and 5%
    scene density, SADMM vs ASADMM on the same seed.  Fixed iteration count
    (the degenerate BASELINE objective meets its stopping rule exactly when the
    screening trigger first fires, so elimination is only
    observable past it).  Reports active-set sizes over the run, the
    compaction / refactor cost, and iterations/s of both modes.  One JSON line
    per density (auxiliary output, not the headline line)."""
    import __graft_entry__
    from paper_2307_08606_b200 import api, scenario
    __graft_entry__.build()
    iters = args.stress_iters
    for which in ("c4_sparse", "c4_dense"):
        cfg = scenario.baseline_config(which)
        s = api.Solver(cfg.N, cfg.Q)
        ys, lam = build_workload(cfg, s, 0, cfg.Q)
        h = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=1e-4, eps_rel=1e-2, max_iter=iters)
        out = {"config": which, "n_targets": cfg.n_targets, "iterations": iters,
               "hyper": {"eps_abs": 1e-4, "eps_rel": 1e-2, "W": 5, "tol": 1e-5, "lambda": lam},
               "warmup": "one untimed ASADMM run of the same problem first (loads the elimination-path "
                         "kernels and sizes the event scratch)"}
        s.run(h, api.Mode.ASADMM, fixed_iterations=True, fetch=False)  # warm-up, untimed
        for mode in (api.Mode.SADMM, api.Mode.ASADMM):
            # timed run as a user runs it (speculation on), then a profiling run
            # of the same solve for the per-phase split (phase events serialise)
            s.set_profiling(False)
            r = s.run(h, mode, fixed_iterations=True)
            ms, _ = s.iteration_stats(r.iterations)
            s.set_profiling(True)
            s.run(h, mode, fixed_iterations=True, fetch=False)
            ph = s.phase_stats()
            s.set_profiling(False)
            trig = next((rec.iteration for rec in r.report.iterations if rec.pri_res <= rec.eps_pri), None)
            sizes = [rec.active_sizes for rec in r.report.iterations]
            ev = [k for k in range(1, len(sizes)) if sizes[k] != sizes[k - 1]]  # 0-based iterations with an event
            quiet = [k for k in range(len(sizes)) if k not in set(ev)]
            ev_ms = float(np.mean([ms[k] for k in ev])) if ev else None
            quiet_ms = float(np.mean([ms[k] for k in quiet])) if quiet else None
            pick = sorted({1, trig or 1, iters // 4, iters // 2, iters})
            out[api.mode_name(mode)] = {
                "iterations_per_s": r.iterations / (float(np.sum(ms)) / 1e3),
                "solve_s_device": float(np.sum(ms)) / 1e3, "setup_s": r.setup_ms / 1e3,
                "first_trigger_iteration": trig, "rebuilds": r.rebuilds, "downdates": r.downdates,
                "active_sizes": {str(k): sizes[k - 1] for k in pick},
                "total_active_solves": r.report.total_active_solves,
                "event_iterations": len(ev), "ms_per_event_iteration": ev_ms, "ms_per_quiet_iteration": quiet_ms,
                "compaction_ms_total": ph["screen"]["ms"], "refactor_ms_total": ph["refactor"]["ms"],
                "phase_ms_note": "compaction/refactor totals from a second, profiled run of the same solve",
                "screen_calls": ph["screen"]["calls"], "refactor_calls": ph["refactor"]["calls"]}
        # time to tolerance (the reference stopping rule, admm.hpp:244-256), both modes
        h_tol = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=1e-4, eps_rel=1e-2, max_iter=3000)
        for mode in (api.Mode.SADMM, api.Mode.ASADMM):
            r = s.run(h_tol, mode)
            ms, _ = s.iteration_stats(r.iterations)
            out[api.mode_name(mode)]["to_tolerance"] = {
                "converged": r.converged, "iterations": r.iterations, "solve_s_device": float(np.sum(ms)) / 1e3,
                "total_active_solves": r.report.total_active_solves,
                "active_sizes_end": r.report.iterations[-1].active_sizes}
        s.close()
        a, p = out["asadmm"], out["sadmm"]
        out["asadmm_vs_sadmm_solve_ratio"] = a["total_active_solves"] / max(1, p["total_active_solves"])
        out["asadmm_vs_sadmm_time_ratio"] = a["solve_s_device"] / max(1e-12, p["solve_s_device"])
        print(json.dumps(out), flush=True)


def frames(args):
    """BASELINE config 5 (multi-frame): the config-2 operators shared by F
    seeded scenes (fresh targets + noise per frame), each solved to the
    time-to-tolerance rule.  Two ways on one resident problem:
      sequential -- one run per frame (the reference's way); the full-set
                    factor is computed once (frame 0) and reused;
      batched    -- run_frames: all frames in lockstep; frames that still
                    share the full active set go through frame-batched DMMA
                    contractions (each operator column read once per
                    iteration for all frames).
    Reports frames/s of both (host wall clock around the solve calls,
    operators already resident) and the per-frame agreement between them.
    One auxiliary JSON line."""
    import __graft_entry__
    from paper_2307_08606_b200 import api, scenario
    from paper_2307_08606_b200.rng import ComplexGaussian, mix_seed
    __graft_entry__.build()
    cfg = scenario.baseline_config("c5")
    s = api.Solver(cfg.N, cfg.Q)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    for q in range(cfg.Q):
        s.generate_dechirp_operator(q, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                    cfg.fc, cfg.bw, cfg.pulse)
    F = args.frames
    ys_all, hypers = [], []
    for f in range(F):
        cfg.frame = f
        xs = scenario.baseline_scene(cfg)
        seed = cfg.seed if f == 0 else mix_seed(cfg.seed, 10000 + f)
        lam = 0.0
        ys = []
        for q in range(cfg.Q):
            y = s.apply(q, xs[q].astype(np.complex128))
            sig = math.sqrt(float(np.vdot(y, y).real) / (cfg.KM * 10.0 ** (cfg.snr_db / 10.0)))
            y = y + sig * ComplexGaussian(mix_seed(seed, q + 1)).draw(cfg.KM)
            ys.append(y)
            lam = max(lam, float(np.abs(s.apply_adjoint(q, y)).max()))
        ys_all.append(ys)
        hypers.append(api.Hyperparams(mu=cfg.mu, lambda_=cfg.lambda_frac * lam, beta=cfg.beta,
                                      eps_abs=cfg.eps_abs, eps_rel=cfg.eps_rel, max_iter=args.ttt_max_iter))
    # the time-to-tolerance rule per frame: eps_abs from that frame's pri_res(1)
    for f in range(F):
        for q in range(cfg.Q):
            s.set_frame_measurement(f, q, ys_all[f][q])
    first = s.run_frames([api.Hyperparams(**{**h.__dict__, "max_iter": 1}) for h in hypers], fetch=True)
    hyp = [api.Hyperparams(**{**h.__dict__, "eps_abs": 1e-5 * r.report.iterations[0].pri_res / math.sqrt(cfg.N)})
           for h, r in zip(hypers, first)]
    # both timed paths start from a cached full-set factor (an untimed
    # 1-iteration run caches the parent's; the frames already hold theirs)
    for q in range(cfg.Q):
        s.set_measurement(q, ys_all[0][q])
    s.run(api.Hyperparams(**{**hyp[0].__dict__, "max_iter": 1}), api.Mode.ASADMM, fetch=False)
    # sequential: one run per frame on the resident problem
    seq = []
    t0 = time.perf_counter()
    for f in range(F):
        for q in range(cfg.Q):
            s.set_measurement(q, ys_all[f][q])
        seq.append(s.run(hyp[f], api.Mode.ASADMM, fetch=False))
    t_seq = time.perf_counter() - t0
    # batched
    t0 = time.perf_counter()
    bat = s.run_frames(hyp, api.Mode.ASADMM, fetch=False)
    t_bat = time.perf_counter() - t0
    # agreement at a FIXED iteration count (to-tolerance runs stop at
    # slightly different iterations, which dominates any end-state diff):
    # batched vs sequential, next to two sequential paths that differ only in
    # fp64 summation order (full vs lower-triangle G-apply) -- the spread the
    # degenerate objective gives any change of rounding.
    kfix = 200
    hfix = [api.Hyperparams(**{**h.__dict__, "max_iter": kfix}) for h in hyp[:2]]
    bfix = s.run_frames(hfix, api.Mode.ASADMM, fixed_iterations=True, fetch=True)
    sfix, sfix0 = [], []
    for f in range(2):
        for q in range(cfg.Q):
            s.set_measurement(q, ys_all[f][q])
        sfix.append(s.run(hfix[f], api.Mode.ASADMM, fixed_iterations=True, fetch=True))
        os.environ["RADMM_HERM"] = "0"
        sfix0.append(s.run(hfix[f], api.Mode.ASADMM, fixed_iterations=True, fetch=True))
        os.environ.pop("RADMM_HERM")
    s.close()
    cat = lambda r: np.concatenate(r.sensor_images)  # noqa: E731
    agree = [api.relative_l2_diff(cat(a), cat(b)) for a, b in zip(bfix, sfix)]
    spread = [api.relative_l2_diff(cat(a), cat(b)) for a, b in zip(sfix0, sfix)]
    iters_seq = [r.iterations for r in seq]
    iters_bat = [r.iterations for r in bat]
    print(json.dumps({"config": "c5", "frames": F,
                      "frames_per_s_sequential": F / t_seq, "frames_per_s_batched": F / t_bat,
                      "speedup_batched": t_seq / t_bat,
                      "wall_s_sequential": t_seq, "wall_s_batched": t_bat,
                      "iterations_per_frame_sequential": iters_seq, "iterations_per_frame_batched": iters_bat,
                      "frame_iterations_per_s_batched": sum(iters_bat) / t_bat,
                      f"sensor_images_rel_diff_at_{kfix}_iterations": {"batched_vs_sequential": max(agree),
                                                                      "summation_order_spread": max(spread)},
                      "converged": all(r.converged for r in bat) and all(r.converged for r in seq),
                      "note": "operators resident; full-set factor computed once and shared; time-to-tolerance "
                              "rule per frame (eps_abs = 1e-5 pri_res(1)/sqrt(N)); wall clock around the solve "
                              "calls; batched = run_frames with frame-batched DMMA contractions"}),
          flush=True)


def spawn_ranks(args) -> bool:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-launch this
    command as N ranks (one process per GPU) through torch.distributed.run on
    127.0.0.1; rank 0 prints the line.  Returns True when it did (the caller
    exits with the launcher's status)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's init lines (nranks) visible in the log
    rc = subprocess.call(cmd, env=env)
    if rc != 0:
        sys.exit(rc)
    return True


def main():
    args = parse()
    if spawn_ranks(args):
        return
    from paper_2307_08606_b200 import scenario
    if args.stress:
        stress(args)
        return
    if args.frames:
        frames(args)
        return
    cfg = scenario.baseline_config(args.config)
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        ours(args, cfg)


if __name__ == "__main__":
    main()
