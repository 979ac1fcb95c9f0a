#!/usr/bin/env python
"""Stage times of repeated config-2 api.run calls from pinned host buffers
(bench.e2e_run's inner loop, every repeat printed): where the slow repeats
lose their time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import bench
    from paper_2307_08606_b200 import api, scenario, distributed as D
    cfg = scenario.baseline_config("c2")
    gen = api.Solver(cfg.N, cfg.Q)
    ys, lam = bench.build_workload(cfg, gen, 0, cfg.Q)
    hyper = api.Hyperparams(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=cfg.eps_abs, eps_rel=cfg.eps_rel,
                            screening_window=5, screening_tol=1e-5, max_iter=3000)
    _, hyper = bench.time_to_tolerance(gen, hyper, 3000)
    buf = api.PinnedBuffer((cfg.Q, cfg.N, cfg.KM), np.complex64)
    for q in range(cfg.Q):
        gen.get_operator_into(q, buf.array[q])
    gen.close()
    ops = [api.ForwardOperator.from_matrix(buf.array[q].T) for q in range(cfg.Q)]
    prob = api.Problem(ops, ys)
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
        r = bench._e2e_once(api, D, torch, prob, hyper, ys, ops, True, 0, cfg.Q, None, 1)
        print(json.dumps({"rep": rep, "it_per_s": round(r["value"], 1), "ms": round(r["ms"], 1),
                          "setup_ms": round(r["setup_ms"], 1), "solve_ms": round(r["solve_ms"], 1),
                          **{k: round(v, 1) for k, v in r["stages_ms"].items()}}), flush=True)
    del prob, ops
    buf.free()


if __name__ == "__main__":
    main()
