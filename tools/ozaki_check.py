#!/usr/bin/env python
"""Ozaki int8 (tcgen05) Gram vs the fp64 DMMA Gram: solves of one C2 sensor's
capacitance system through each, against each other and the exact inverse."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2307_08606_b200 import api, scenario
    cfg = scenario.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
    s = api.Solver(cfg.N, 1)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    s.generate_dechirp_operator(0, cfg.M, cfg.K, pix, tx[0], rx[0], scenario.baseline_phases(cfg, 0),
                                cfg.fc, cfg.bw, cfg.pulse)
    a = s.get_operator(0).astype(np.complex128)
    s.close()
    rng = np.random.default_rng(1)
    rhs = [rng.normal(size=cfg.N) + 1j * rng.normal(size=cfg.N) for _ in range(3)]
    out = {}
    for flag in ("0", "1"):
        os.environ["RADMM_OZAKI"] = flag
        t0 = time.perf_counter()
        cache = api.factorize(a, 1.0, 1.0)
        t1 = time.perf_counter()
        out[flag] = [cache.solve(r) for r in rhs]
        print(f"RADMM_OZAKI={flag}: factorize {1e3 * (t1 - t0):.1f} ms (host wall, incl. upload)", flush=True)
    for i, r in enumerate(rhs):
        d = np.linalg.norm(out["1"][i] - out["0"][i]) / np.linalg.norm(out["0"][i])
        print(f"rhs {i}: ozaki vs dmma solve rel diff {d:.3e}")


if __name__ == "__main__":
    main()
