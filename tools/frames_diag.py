#!/usr/bin/env python
"""Diagnostic (GPU): batched frames vs separate runs at config-2 size, per
iteration count, with and without the batched contractions."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_08606_b200 import api, scenario  # noqa: E402

cfg = scenario.baseline_config("c2")
s = api.Solver(cfg.N, cfg.Q)
pix, tx, rx = scenario.baseline_geometry(cfg)
for q in range(cfg.Q):
    s.generate_dechirp_operator(q, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                cfg.fc, cfg.bw, cfg.pulse)
xs = scenario.baseline_scene(cfg)
ys = [s.apply(q, xs[q].astype(np.complex128)) for q in range(cfg.Q)]
rng = np.random.default_rng(5)
frames = [ys, [y + 1e-3 * (rng.normal(size=y.shape) + 1j * rng.normal(size=y.shape)) for y in ys]]
for f, yf in enumerate(frames):
    for q in range(cfg.Q):
        s.set_frame_measurement(f, q, yf[q])


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


for batch in ("1", "0"):
    os.environ["RADMM_FRAME_BATCH"] = batch
    for it in (1, 2, 5, 10):
        h = api.Hyperparams(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=it)
        res = s.run_frames([h, h], api.Mode.ASADMM, fixed_iterations=True)
        out = []
        for f, yf in enumerate(frames):
            for q in range(cfg.Q):
                s.set_measurement(q, yf[q])
            one = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
            out.append((rel(np.concatenate(res[f].sensor_images), np.concatenate(one.sensor_images)),
                        rel(res[f].sigma, one.sigma), rel(res[f].s, one.s)))
        print(f"batch={batch} iters={it}:", ["img %.2e sig %.2e s %.2e" % o for o in out], flush=True)
os.environ["RADMM_HERM"] = "0"
for it in (1, 2, 5, 10):  # summation-order spread of the plain path
    h = api.Hyperparams(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=it)
    out = []
    for f, yf in enumerate(frames):
        for q in range(cfg.Q):
            s.set_measurement(q, yf[q])
        os.environ["RADMM_HERM"] = "0"
        a = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
        os.environ["RADMM_HERM"] = "1"
        b = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
        out.append((rel(np.concatenate(a.sensor_images), np.concatenate(b.sensor_images)), rel(a.sigma, b.sigma),
                    rel(a.s, b.s)))
    print(f"herm0 vs herm1 iters={it}:", ["img %.2e sig %.2e s %.2e" % o for o in out], flush=True)
