#!/usr/bin/env python
"""Where the end-to-end time of one api.run call goes (C2 by default).

    python tools/e2e_breakdown.py [--config c2] [--fixed 25]

Stages, host wall clock with the context stream synchronised by each ABI
call: context create, per-sensor operator upload (pinned host -> HBM),
measurements, the run (its own setup_ms / solve_ms split), result fetch,
context destroy.  One JSON line.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--fixed", type=int, default=0, help="fixed iteration count (0: to tolerance)")
    ap.add_argument("--q", type=int, default=0, help="override the sensor count (setup probes at config-3 shapes)")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2307_08606_b200 import api, scenario
    cfg = scenario.baseline_config(a.config, **({"Q": a.q} if a.q else {}))
    gen = api.Solver(cfg.N, cfg.Q)
    ys, lam = bench.build_workload(cfg, gen, 0, cfg.Q)
    hyper = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=cfg.eps_abs, eps_rel=cfg.eps_rel,
                            screening_window=5, screening_tol=1e-5, max_iter=a.fixed or 3000)
    if not a.fixed:
        _, hyper = bench.time_to_tolerance(gen, hyper, 3000)
    pinned = torch.empty((cfg.Q, cfg.N, cfg.KM), dtype=torch.complex64, pin_memory=True)
    for q in range(cfg.Q):
        pinned[q].numpy()[:] = gen.get_operator(q).T
    gen.close()
    mats = [pinned[q].numpy().T for q in range(cfg.Q)]
    out = {"config": a.config}
    t = time.perf_counter()
    s = api.Solver(cfg.N, cfg.Q)
    out["ctx_create_ms"] = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter()
    for q in range(cfg.Q):
        s.set_operator(q, mats[q])
    dt = time.perf_counter() - t
    out["operator_upload_ms"] = 1e3 * dt
    out["operator_upload_GBps"] = sum(m.nbytes for m in mats) / dt / 1e9
    t = time.perf_counter()
    for q in range(cfg.Q):
        s.set_measurement(q, ys[q])
    out["measurement_ms"] = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter()
    r = s.run(hyper, api.Mode.ASADMM, fixed_iterations=bool(a.fixed), fetch=False)
    out["run_ms"] = 1e3 * (time.perf_counter() - t)
    out["setup_ms"], out["solve_ms"], out["iterations"] = r.setup_ms, r.solve_ms, r.iterations
    t = time.perf_counter()
    s._fetch(r)
    out["fetch_ms"] = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter()
    s.close()
    out["destroy_ms"] = 1e3 * (time.perf_counter() - t)
    out["phase_note"] = "setup = initial data terms + Gram + Gauss-Jordan inverse (see DESIGN.md section 3)"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
