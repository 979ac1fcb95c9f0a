import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2307_08606_b200 import api, scenario
cfg = scenario.baseline_config("c4_sparse")
s = api.Solver(cfg.N, cfg.Q)
ys, lam = bench.build_workload(cfg, s, 0, cfg.Q)
h = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=1e-4, eps_rel=1e-2, max_iter=400)
for rep in range(3):
    r = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
    ms, ln = s.iteration_stats(r.iterations)
    ms = np.asarray(ms)
    print(f"run {rep}: total {ms.sum():.1f} ms, median {np.median(ms):.3f}, max {ms.max():.3f}, iterations > 1.5 ms: {(ms > 1.5).sum()}, launches {int(np.sum(ln))}", flush=True)
    if rep == 0:
        print("slowest iterations:", np.argsort(ms)[-8:] + 1, np.sort(ms)[-8:])
