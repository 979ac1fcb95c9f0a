#!/usr/bin/env python
"""Diagnostic (GPU): accuracy of the G-apply variants (RADMM_HERM 0/1/2) with
and without the Hermitian projection of the factor (RADMM_SYMM 0/1): dual
solves on the C1 operator against the exact solve, and the C1 300-iteration
run against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2307_08606_b200 import api, scenario  # noqa: E402
from _parity import gpu_run, oracle_run, state_errors  # noqa: E402

cfg = scenario.baseline_config("c1")
a = scenario.baseline_operator(cfg, 0).astype(np.complex128)
aq = a.astype(np.complex64).astype(np.complex128)
cap = np.eye(a.shape[0]) + aq @ aq.conj().T
rng = np.random.default_rng(0)
rhs = [rng.normal(size=a.shape[1]) + 1j * rng.normal(size=a.shape[1]) for _ in range(3)]
refs = [r - aq.conj().T @ np.linalg.solve(cap, aq @ r) for r in rhs]
ops, ys, _, hyper = scenario.baseline_problem(cfg)
o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
for symm in ("0", "1"):
    for herm in ("0", "1", "2"):
        os.environ["RADMM_SYMM"], os.environ["RADMM_HERM"] = symm, herm
        cache = api.factorize(a, 1.0, 1.0)
        err = max(np.linalg.norm(cache.solve(r) - f) / np.linalg.norm(f) for r, f in zip(rhs, refs))
        g = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
        e = state_errors(g, o)
        print(f"SYMM={symm} HERM={herm}: c1 solve rel err {err:.3e}; 300-it vs oracle: "
              + ", ".join(f"{k} {v:.2e}" for k, v in e.items()), flush=True)
