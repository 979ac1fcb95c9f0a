#!/usr/bin/env python
"""Per-sensor host time of radmm_set_operator_c64 at config-3 size from pinned
host memory, with and without the eager Gram behind each upload.

    python tools/upload_probe.py [--sensors 6]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sensors", type=int, default=6)
    ap.add_argument("--ctx-sensors", type=int, default=32, help="sensors the context is created for")
    a = ap.parse_args()
    import torch
    from paper_2307_08606_b200 import api, scenario
    cfg = scenario.baseline_config("c3")
    Q = a.sensors
    buf = api.PinnedBuffer((Q, cfg.N, cfg.KM), np.complex64)
    gen = api.Solver(cfg.N, 1)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    for q in range(Q):
        gen.generate_dechirp_operator(0, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                      cfg.fc, cfg.bw, cfg.pulse)
        gen.get_operator_into(0, buf.array[q])
    gen.close()
    for eager in ("1", "0"):
        api.set_tuning("RADMM_EAGER_GRAM", int(eager))
        s = api.Solver(cfg.N, max(Q, a.ctx_sensors))
        ts = []
        for q in range(Q):
            t0 = time.perf_counter()
            s.set_operator(q, buf.array[q].T)
            ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        torch.cuda.synchronize()
        tail = time.perf_counter() - t0
        print(f"eager={eager}: set_operator per sensor (s): {[round(t, 3) for t in ts]}, device tail {tail:.3f} s",
              flush=True)
        s.close()
    api.set_tuning("RADMM_EAGER_GRAM", None)


if __name__ == "__main__":
    main()
