"""One elimination-stress run (config-4 geometry) for profiling the event path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2307_08606_b200 import api, scenario
which, iters = sys.argv[1], int(sys.argv[2])
cfg = scenario.baseline_config(which)
s = api.Solver(cfg.N, cfg.Q)
ys, lam = bench.build_workload(cfg, s, 0, cfg.Q)
h = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=1e-4, eps_rel=1e-2, max_iter=iters)
r = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
print("rebuilds", r.rebuilds, "downdates", r.downdates, "removal log", len(r.removal_log))
import collections
per = collections.Counter((int(k), int(q)) for k, q, _ in r.removal_log)
print("events (iteration, sensor):", len(per), "max removed in one", max(per.values()) if per else 0)
