#!/usr/bin/env python
"""Generate the committed full-size oracle fixtures (tests/golden/*.npz).

The fp64 CPU oracle (oracle/admm_ref.py) runs here, once, on the BASELINE
workloads at their full sizes; the GPU parity tests (tests/test_gpu_fixtures.py,
``-m gpu``) replay the same inputs through the C ABI and compare.  Inputs are
bit-identical on both sides: the operators come from the portable generator
(scenario.baseline_operator == radmm_generate_dechirp_operator bit for bit; a
SHA-256 of every sensor's complex64 operator is stored and checked on the GPU
box), and the measurements y and lambda are stored in the fixture.

    python tests/golden/gen_parity_fixtures.py [c2_fixed c2_ttt c4_masks c3_q2 c5_frames lambdas]

Cost here (8 cores): c2_fixed ~2 min, c2_ttt ~23 min, c4_masks ~5 min,
c3_q2 ~10 min, c5_frames ~5 min, lambdas ~5 min.
"""
from __future__ import annotations

import hashlib
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import admm_ref  # noqa: E402
from paper_2307_08606_b200 import scenario  # noqa: E402


def op_digest(a64: np.ndarray) -> str:
    """SHA-256 of a sensor operator, complex64, column-major (pixel columns
    contiguous) -- the layout radmm_get_operator_c64 returns."""
    return hashlib.sha256(np.asfortranarray(a64).tobytes(order="F")).hexdigest()


def problem(cfg, q_count=None):
    """Host operators (portable generator), seeded scene, measurements, lambda."""
    from oracle import gen  # the C host generator: bitwise scenario.baseline_operator, ~100x faster
    q_count = q_count or cfg.Q
    ops = [gen.baseline_operator(cfg, q) for q in range(q_count)]
    per_sensor = scenario.baseline_scene(cfg)[:q_count]
    ys = scenario.baseline_measurements(cfg, ops, per_sensor)
    lam = scenario.baseline_lambda(cfg, ops, ys)
    return ops, ys, lam


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


def records(res):
    return np.array([[r.pri_res, r.dual_res, r.eps_pri, r.eps_dual] for r in res.records])


def common(cfg, ops, ys, lam, hyper):
    return dict(digests=np.array([op_digest(a) for a in ops]), ys=np.stack(ys), lam=np.float64(lam),
                hyper=np.array([hyper["mu"], hyper["lambda_"], hyper["beta"], hyper["eps_abs"], hyper["eps_rel"],
                                hyper["screening_window"], hyper["screening_tol"], hyper["max_iter"]]),
                cfg=np.array([cfg.name, str(cfg.Q), str(cfg.M), str(cfg.K), str(cfg.nside), str(cfg.frame)]))


def gen_c2_fixed(iters=100):
    """BASELINE config 2, full size, the bench's lambda, `iters` fixed iterations."""
    cfg = scenario.baseline_config("c2")
    ops, ys, lam = problem(cfg)
    hyper = scenario.baseline_hyper(cfg, lam)
    hyper["max_iter"] = iters
    t0 = time.time()
    o = admm_ref.run(ops, ys, admm_ref.Hyper(**hyper), asadmm=True, fixed_iterations=True)
    print(f"c2_fixed: {o.iterations} iterations in {time.time() - t0:.0f} s", flush=True)
    save("c2_fixed", **common(cfg, ops, ys, lam, hyper), records=records(o),
         sensor_images=np.stack(o.sensor_images).astype(np.complex64), s=o.s, sigma=o.sigma,
         sizes=np.array([r.active_sizes for r in o.records]))


def gen_c2_ttt():
    """BASELINE config 2 to tolerance with the bench's rule
    (eps_abs = 1e-5 pri_res(1) / sqrt(N), eps_rel = 1e-5): stopping iteration
    and the pri/dual/eps traces."""
    cfg = scenario.baseline_config("c2")
    ops, ys, lam = problem(cfg)
    hyper = scenario.baseline_hyper(cfg, lam)
    first = admm_ref.run(ops, ys, admm_ref.Hyper(**{**hyper, "max_iter": 1}), asadmm=True)
    hyper["eps_abs"] = 1e-5 * first.records[0].pri_res / math.sqrt(cfg.N)
    hyper["max_iter"] = 3000
    t0 = time.time()
    o = admm_ref.run(ops, ys, admm_ref.Hyper(**hyper), asadmm=True)
    print(f"c2_ttt: converged={o.converged} after {o.iterations} iterations in {time.time() - t0:.0f} s",
          flush=True)
    save("c2_ttt", **common(cfg, ops, ys, lam, hyper), records=records(o), iterations=np.int64(o.iterations),
         converged=np.bool_(o.converged), sizes=np.array([r.active_sizes for r in o.records]))


def event_arrays(o, tol):
    """Per screening step (k, q): removed pixels, and the pixels whose oracle
    criterion lies within a relative 1e-6 of the tolerance (near-threshold)."""
    keys, removed, near = [], [], []
    for e in o.events:
        if e.zeta is None:
            continue
        keys.append((e.iteration, e.sensor))
        removed.append(np.sort(e.removed))
        band = np.abs(e.zeta - tol) <= 1e-6 * tol
        near.append(np.sort(e.active_before[band]))
    flat = lambda lists: (np.concatenate(lists) if lists else np.zeros(0, np.int64),  # noqa: E731
                          np.cumsum([0] + [len(x) for x in lists]))
    rv, ro = flat(removed)
    nv, no = flat(near)
    return dict(ev_keys=np.array(keys, dtype=np.int64).reshape(-1, 2), ev_removed=rv, ev_removed_off=ro,
                ev_near=nv, ev_near_off=no)


def gen_c4_masks(q_count=4, past_trigger=40):
    """BASELINE config 4 (sparse: 0.1% of pixels) at config-2 geometry with
    Q reduced to `q_count`, the reference's default tolerances so the
    screening trigger fires, `past_trigger` iterations past the first
    trigger: elimination masks at every step."""
    cfg = scenario.baseline_config("c4_sparse", Q=q_count, eps_abs=1e-4, eps_rel=1e-2)
    ops, ys, lam = problem(cfg)
    hyper = scenario.baseline_hyper(cfg, lam)
    probe = admm_ref.run(ops, ys, admm_ref.Hyper(**{**hyper, "max_iter": 200}), asadmm=False, fixed_iterations=True)
    trig = next(r.iteration for r in probe.records if r.pri_res <= r.eps_pri)
    hyper["max_iter"] = trig + past_trigger
    t0 = time.time()
    o = admm_ref.run(ops, ys, admm_ref.Hyper(**hyper), asadmm=True, fixed_iterations=True)
    print(f"c4_masks: trigger at {trig}, {o.iterations} iterations in {time.time() - t0:.0f} s, "
          f"final sizes {o.records[-1].active_sizes}", flush=True)
    save("c4_masks", **common(cfg, ops, ys, lam, hyper), records=records(o), trigger=np.int64(trig),
         sizes=np.array([r.active_sizes for r in o.records]),
         sensor_images=np.stack(o.sensor_images).astype(np.complex64), s=o.s, sigma=o.sigma,
         **event_arrays(o, hyper["screening_tol"]))


def gen_c3_q2(iters=5):
    """BASELINE config 3 shapes (KM = 8192, N = 65536) with Q reduced to 2."""
    cfg = scenario.baseline_config("c3")
    q_count = 2
    t0 = time.time()
    ops, ys, lam = problem(cfg, q_count)
    print(f"c3_q2: inputs in {time.time() - t0:.0f} s", flush=True)
    hyper = scenario.baseline_hyper(cfg, lam)
    hyper["max_iter"] = iters
    t0 = time.time()
    o = admm_ref.run(ops, ys, admm_ref.Hyper(**hyper), asadmm=True, fixed_iterations=True)
    print(f"c3_q2: {o.iterations} iterations in {time.time() - t0:.0f} s", flush=True)
    save("c3_q2", **common(cfg, ops, ys, lam, hyper), records=records(o),
         sensor_images=np.stack(o.sensor_images).astype(np.complex64), s=o.s, sigma=o.sigma)


def gen_c5_frames(frames=(1, 2), iters=100):
    """BASELINE config 5: frames of the config-2 operator (fresh targets and
    noise per frame), `iters` fixed iterations each -- the reference's
    sequential per-frame runs; the GPU's batched run_frames is compared."""
    cfg0 = scenario.baseline_config("c5")
    ops = [scenario.baseline_operator(cfg0, q) for q in range(cfg0.Q)]
    out = {}
    for f in frames:
        cfg = scenario.baseline_config("c5", frame=f)
        per_sensor = scenario.baseline_scene(cfg)
        ys = scenario.baseline_measurements(cfg, ops, per_sensor)
        lam = scenario.baseline_lambda(cfg, ops, ys)
        hyper = scenario.baseline_hyper(cfg, lam)
        hyper["max_iter"] = iters
        t0 = time.time()
        o = admm_ref.run(ops, ys, admm_ref.Hyper(**hyper), asadmm=True, fixed_iterations=True)
        print(f"c5 frame {f}: {o.iterations} iterations in {time.time() - t0:.0f} s", flush=True)
        out[f"f{f}_ys"] = np.stack(ys)
        out[f"f{f}_lam"] = np.float64(lam)
        out[f"f{f}_records"] = records(o)
        out[f"f{f}_sensor_images"] = np.stack(o.sensor_images).astype(np.complex64)
        out[f"f{f}_s"] = o.s
        out[f"f{f}_sigma"] = o.sigma
    save("c5_frames", digests=np.array([op_digest(a) for a in ops]), frames=np.array(frames),
         iters=np.int64(iters), **out)


def gen_lambdas():
    """lambda = 0.05 max_q |A_q^H y_q|_inf of every BASELINE config (host
    generator): the reference arm of bench.py prints the same lambda as the
    GPU arm without regenerating all 32 config-3 operators (~2 min)."""
    import json
    from oracle import gen
    out = {}
    for name in ("c1", "c2", "c3", "c4_sparse", "c4_dense"):
        cfg = scenario.baseline_config(name)
        per_sensor = scenario.baseline_scene(cfg)
        m = 0.0
        for q in range(cfg.Q):
            a = gen.baseline_operator(cfg, q)
            y = scenario.simulate_measurement(a, per_sensor[q], cfg.snr_db, scenario.mix_seed(cfg.seed, q + 1))[0]
            m = max(m, float(np.abs(a.conj().T @ y).max()))
        out[name] = cfg.lambda_frac * m
        print(name, out[name], flush=True)
    with open(os.path.join(HERE, "baseline_lambdas.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    jobs = sys.argv[1:] or ["c2_fixed", "c2_ttt", "c4_masks", "c5_frames", "c3_q2"]
    for j in jobs:
        globals()["gen_" + j]()
