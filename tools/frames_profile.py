#!/usr/bin/env python
"""Per-pass device time of the frame-batched contractions (BASELINE config 5
shapes): F frames x 8 sensors, fixed iterations, profiling on.  Prints the
average ms per call of the batched forward / G-apply / adjoint passes and
the achieved fp64 TFLOP/s of each (8 real flops per complex multiply-add)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=16)
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    from paper_2307_08606_b200 import api, scenario
    from paper_2307_08606_b200.rng import ComplexGaussian, mix_seed
    cfg = scenario.baseline_config("c5")
    s = api.Solver(cfg.N, cfg.Q)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    for q in range(cfg.Q):
        s.generate_dechirp_operator(q, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                    cfg.fc, cfg.bw, cfg.pulse)
    hyp = []
    for f in range(a.frames):
        cfg.frame = f
        xs = scenario.baseline_scene(cfg)
        for q in range(cfg.Q):
            y = s.apply(q, xs[q].astype(np.complex128))
            y = y + 1e-3 * ComplexGaussian(mix_seed(7, 100 * f + q)).draw(cfg.KM)
            s.set_frame_measurement(f, q, y)
        hyp.append(api.Hyperparams(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=a.iters))
    s.run_frames(hyp, fixed_iterations=True, fetch=False)  # warm
    s.set_profiling(True)
    s.run_frames(hyp, fixed_iterations=True, fetch=False)
    ph = s.phase_stats()
    F, Q, KM, N = a.frames, cfg.Q, cfg.KM, cfg.N
    flops = {"forward": 8.0 * Q * KM * N * F, "adjoint": 8.0 * Q * KM * N * F, "gapply": 8.0 * Q * KM * KM * F}
    out = {"frames": F, "iterations": a.iters}
    for k in ("forward", "gapply", "adjoint"):
        st = ph[k]
        ms = st["ms"] / max(1, st["calls"])
        out[k] = {"ms_per_call": ms, "tflops": flops[k] / ms / 1e9 if ms > 0 else None, "calls": st["calls"]}
    s.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
