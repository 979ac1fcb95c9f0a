import time, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2307_08606_b200 import api, scenario
cfg = scenario.baseline_config("c2")
out = []
keep = api.Solver(cfg.N, cfg.Q)
ys, lam = bench.build_workload(cfg, keep, 0, cfg.Q)
h = api.Hyperparams(mu=1.0, lambda_=lam, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=5)
ops = [keep.get_operator(q) for q in range(cfg.Q)]
for rep in range(4):
    t0 = time.perf_counter(); s = api.Solver(cfg.N, cfg.Q)
    for q in range(cfg.Q):
        s.set_operator(q, ops[q]); s.set_measurement(q, ys[q])
    t1 = time.perf_counter(); r = s.run(h, fixed_iterations=True, fetch=True); t2 = time.perf_counter()
    s.close(); t3 = time.perf_counter()
    out.append({"create_upload": round(1e3*(t1-t0),1), "run": round(1e3*(t2-t1),1), "close": round(1e3*(t3-t2),1), "setup": round(r.setup_ms,1)})
print(json.dumps(out))
