#!/usr/bin/env python
"""GPU vs fp64 oracle on BASELINE config 2 at full size, iteration by
iteration (diagnostic for tests/test_gpu_parity.py's full-size parity).

    python tools/c2_oracle_diag.py [--iters 3]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    from oracle import admm_ref
    from paper_2307_08606_b200 import api, scenario
    cfg = scenario.baseline_config(a.config)
    s = api.Solver(cfg.N, cfg.Q)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    for q in range(cfg.Q):
        s.generate_dechirp_operator(q, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                    cfg.fc, cfg.bw, cfg.pulse)
    xs = scenario.baseline_scene(cfg)
    ys = [s.apply(q, xs[q].astype(np.complex128)) for q in range(cfg.Q)]
    for q, y in enumerate(ys):
        s.set_measurement(q, y)
    ops = [s.get_operator(q).astype(np.complex128) for q in range(cfg.Q)]
    rel = lambda x, y: float(np.linalg.norm(np.ravel(x) - np.ravel(y)) / max(1e-300, np.linalg.norm(np.ravel(y))))
    for it in range(1, a.iters + 1):
        hyper = dict(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=it)
        g = s.run(api.Hyperparams(**hyper), api.Mode.ASADMM, fixed_iterations=True)
        o = admm_ref.run(ops, ys, admm_ref.Hyper(**hyper), asadmm=True, fixed_iterations=True)
        per_q = [rel(g.sensor_images[q], o.sensor_images[q]) for q in range(cfg.Q)]
        print(f"iters={it}: sensor images {rel(np.concatenate(g.sensor_images), np.concatenate(o.sensor_images)):.3e} "
              f"(per sensor max {max(per_q):.3e}), s {rel(g.s, o.s):.3e}, sigma {rel(g.sigma, o.sigma):.3e}, "
              f"pri {g.report.iterations[-1].pri_res:.6e} vs {o.records[-1].pri_res:.6e}", flush=True)
    s.close()


if __name__ == "__main__":
    main()
