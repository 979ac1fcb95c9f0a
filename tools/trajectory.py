"""Print the C2 convergence trajectory (pri/dual residuals vs tolerances, active sizes)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2307_08606_b200 import api, scenario

cfg = scenario.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
eps_abs = float(sys.argv[3]) if len(sys.argv) > 3 else cfg.eps_abs
s = api.Solver(cfg.N, cfg.Q)
ys, lam = bench.build_workload(cfg, s, 0, cfg.Q)
h = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=eps_abs, eps_rel=cfg.eps_rel, max_iter=iters)
r = s.run(h, api.Mode.ASADMM)
wall, _ = s.iteration_stats(r.iterations)
print("converged", r.converged, "iterations", r.iterations, "setup_ms", r.setup_ms, "rebuilds", r.rebuilds,
      "downdates", r.downdates, "solve_ms(host)", r.solve_ms, "device wall ms", wall.sum())
for rec in r.report.iterations:
    if rec.iteration in (1, 2, 5, 10, 20, 50, 100, 200, 300, 500, 1000, 1500, 2000, 2500, 3000) or rec is r.report.iterations[-1]:
        print(rec.iteration, "pri %.3e eps_pri %.3e dual %.3e eps_dual %.3e" % (rec.pri_res, rec.eps_pri, rec.dual_res, rec.eps_dual),
              "act", rec.active_sizes, "ms %.3f" % wall[rec.iteration - 1])
print("|x_G|", np.linalg.norm(r.x_global), "|s|", np.linalg.norm(r.s))
