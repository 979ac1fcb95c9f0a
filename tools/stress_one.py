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
ms_asadmm, _ = s.iteration_stats(r.iterations)
print("rebuilds", r.rebuilds, "downdates", r.downdates, "removal log", len(r.removal_log))
import collections
per = collections.Counter((int(k), int(q)) for k, q, _ in r.removal_log)
print("events (iteration, sensor):", len(per), "max removed in one", max(per.values()) if per else 0)
# how much a multi-RHS G-apply / device-resident events could cover
hist = collections.Counter(per.values())
print("removed per (iteration, sensor):", dict(sorted(hist.items())))
by_it = collections.defaultdict(list)
for (k, q), n in per.items():
    by_it[k].append(n)
mx = collections.Counter(max(v) for v in by_it.values())
print("event iterations:", len(by_it), "max removed over sensors per event iteration:", dict(sorted(mx.items())))
import numpy as np
ms = np.asarray(ms_asadmm)
if ms is not None and len(ms):
    ev = np.zeros(len(ms), bool)
    for k in by_it:
        if 1 <= k <= len(ms):
            ev[k - 1] = True
    print(f"iteration ms: event {ms[ev].mean():.4f} (n={ev.sum()}), quiet {ms[~ev].mean():.4f} (n={(~ev).sum()}), total {ms.sum():.2f}")
r2 = s.run(h, api.Mode.SADMM, fixed_iterations=True)
ms2, _ = s.iteration_stats(r2.iterations)
print(f"SADMM total {np.sum(ms2):.2f} ms; ASADMM/SADMM {ms.sum() / np.sum(ms2):.3f}")
