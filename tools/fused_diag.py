#!/usr/bin/env python
"""Diagnostic (GPU): state after k iterations for RADMM_FUSED = 0 / 4 / 5."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2307_08606_b200 import api, scenario  # noqa: E402

cfg = scenario.baseline_config("c1", nside=32, K=64, M=8, n_targets=6, max_iter=3)
ops, ys, _, hyper = scenario.baseline_problem(cfg)
hyper = dict(hyper, screening_tol=1e-3)


def run(v, it):
    os.environ["RADMM_FUSED"] = v
    prob = api.Problem([api.ForwardOperator.from_matrix(a) for a in ops], ys)
    r = api.run(prob, api.Hyperparams(**dict(hyper, max_iter=it)), api.Mode.ASADMM, fixed_iterations=True)
    return r


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


for it in (1, 2, 3):
    base = run("0", it)
    for v in ("4", "5"):
        r = run(v, it)
        per = [rel(x, y) for x, y in zip(r.sensor_images, base.sensor_images)]
        print(f"it={it} v{v}: sensor_images {['%.1e' % p for p in per]} s {rel(r.s, base.s):.1e} "
              f"sigma {rel(r.sigma, base.sigma):.1e} pri {r.report.iterations[-1].pri_res:.6e} "
              f"vs {base.report.iterations[-1].pri_res:.6e}", flush=True)
